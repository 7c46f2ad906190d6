"""A CPU model of the kernels' index algorithm, driven by the REAL launch descriptor.

triot_plan_describe() returns the descriptor the library would pass to the sm_100a kernel
(canonical digits, +32-vector step digits, per-tensor strides and carry deltas, bounds).
This model runs exactly the kernel's per-lane algorithm on it -- decode the start vector,
then advance +32 vectors with the unrolled carry loop, adding the carry deltas to each
tensor's offset -- and applies the op on numpy buffers.  Comparing its output with the oracle
on small random shapes checks the host plan (validation, canonicalisation, vector geometry,
carry deltas) without a GPU.  It is a test helper: the product never runs it.
"""
from __future__ import annotations

import numpy as np

M32 = (1 << 32) - 1


def _wrap(x, idx64):
    return x if idx64 else (x & M32)


def run_ev_rows(desc: dict, p):
    """The dense EV's shared-memory row tiles (ev_rows_kernel): rows of rowlen elements, the
    outer digits of row index r (decoded over `ext`) weight the row's mass, the column moment
    goes to slot D, the mass to slot D + 1 -- checks the plan's digits and slot mapping."""
    D, ext, n = desc["D"], desc["ext"], desc["rowlen"]
    slots = [0.0] * (D + 2)
    for r in range(desc["nvec"]):
        row = p[r * n:(r + 1) * n]
        u, v = [0] * D, r
        for k in range(D - 1, 0, -1):
            u[k] = v % ext[k]
            v //= ext[k]
        u[0] = v
        mass = float(np.sum(row, dtype=np.float64))
        for k in range(D):
            slots[k] += u[k] * mass
        slots[D] += float(sum(c * float(row[c]) for c in range(n)))
        slots[D + 1] += mass
    d = desc["d"]
    return [slots[sl] if sl >= 0 else 0.0 for sl in desc["slot_of_axis"][:d]]


def run(desc: dict, op: str, bufs: list, binop: str = "mul"):
    """bufs: flat numpy arrays in tensor order (embed: dst, src; binary: c, a, b; ev: p).
    Writes outputs in place; for 'ev' returns the weight-slot totals (list of floats)."""
    if op == "ev" and desc.get("evrows"):
        return run_ev_rows(desc, bufs[0])
    D, V, idx64 = desc["D"], desc["V"], desc["idx64"]
    ext, dlt, bnd = desc["ext"], desc["dlt"], desc["bnd"]
    khi, klo, lgL = desc["khi"], desc["klo"], desc["lgL"]
    T = desc["t"]
    nt = len(T)
    L = 1 << lgL
    nvec = desc["nvec"]
    W = lambda x: _wrap(x, idx64)
    slots = [0.0] * (D + 1)

    def start(v):
        v0 = v
        u = [0] * D
        for k in range(D - 1, 0, -1):
            u[k] = v % ext[k]
            v //= ext[k]
        u[0] = v
        off = [W(sum(u[k] * T[x]["sig"][k] for k in range(D))) for x in range(nt)]
        if desc.get("lin0"):   # the kernel's shortcut for a tensor 0 dense in the digit space
            assert off[0] == W(v0 * desc["lin0"]), (off[0], v0, desc["lin0"])
        oob = 0
        for k in range(D - 1):
            oob |= int(u[k] >= bnd[k]) << k
        return u, off, oob

    def step(u, off, oob):
        off = [W(off[x] + T[x]["step"]) for x in range(nt)]
        carry = 0
        for k in range(D - 1, -1, -1):
            if k > khi:
                continue
            nu = u[k] + dlt[k] + carry
            carry = int(nu >= ext[k])
            if carry:
                nu -= ext[k]
                off = [W(off[x] + T[x]["kap"][k]) for x in range(nt)]
            u[k] = nu
            if k < D - 1:
                oob = (oob & ~(1 << k)) | (int(nu >= bnd[k]) << k)
            if k <= klo and not carry:
                break
        return u, off, oob

    def eoff(x, off, e):
        r, c = e >> lgL, e & (L - 1)
        return W(off + r * T[x]["rho"] + c * T[x]["tau"])

    if desc.get("flat"):
        return run_flat(desc, op, bufs, binop)
    if desc.get("rows"):
        return run_rows(desc, op, bufs, binop)
    wmul, wspan, dv = desc["wmul"], desc["wspan"], desc["dv"]
    # mode 0: warp chunks; 1: grid stride; 2: block chunks, thread t starts at vector t
    if desc["mode"] == 2:
        units, lanes = (nvec + wmul - 1) // wmul, dv
    else:
        units = (nvec + wmul - 1) // wmul if desc["mode"] == 0 else dv // 32
        lanes = 32
    for w in range(units):
        base0 = w * wmul
        if base0 >= nvec:
            continue
        vend = min(base0 + wspan, nvec)
        for lane in range(lanes):
            v = base0 + lane
            u, off, oob = start(v)
            zmask = desc.get("zmask", 0)
            while v < vend:
                if op == "embed" and oob & zmask:
                    # zero run: digit m stays out of bounds until digits m..khi wrap
                    m = ((oob & zmask) & -(oob & zmask)).bit_length() - 1
                    S, N = 0, 1
                    for k in range(m, khi + 1):
                        S, N = S * ext[k] + u[k], N * ext[k]
                    # the kernel's form: N from the plan, S = (step index) mod N
                    T_ = (v - lane) // 32
                    assert desc["zn"][m] == N and T_ % N == S, (desc["zn"], m, N, S, T_)
                    run_ = min(N - S, (vend - (v - lane) + 31) // 32)
                    o = off[0]
                    for r in range(run_):
                        if v + 32 * r < vend:
                            for e in range(V):
                                bufs[0][eoff(0, o, e)] = 0
                        o = W(o + T[0]["step"])
                    v += 32 * run_
                    if v < vend:
                        # the kernel's carry instead of a re-decode: digits m..khi restart at 0,
                        # digit m-1 takes the carry; must equal the decoded tuple of v
                        nu_ = list(u)
                        for k in range(m, khi + 1):
                            nu_[k] = 0
                        for k in range(m - 1, -1, -1):
                            nu_[k] += 1
                            if k > 0 and nu_[k] >= ext[k]:
                                nu_[k] = 0
                                continue
                            break
                        u, off, oob = start(v)
                        assert nu_ == u, (nu_, u)
                    continue
                if True:
                    uv = u[D - 1]
                    if op == "embed":
                        vals = np.zeros(V, dtype=bufs[0].dtype)
                        anyb = oob == 0 and uv < desc["vany"]
                        if anyb and uv < desc["vfull"]:
                            vals = np.array([bufs[1][eoff(1, off[1], e)] for e in range(V)],
                                            dtype=bufs[0].dtype)
                        elif anyb:
                            row0, col0 = uv * desc["rowmul"], uv * desc["colmul"]
                            for e in range(V):
                                r, c = e >> lgL, e & (L - 1)
                                if row0 + r < desc["srows"] and col0 + c < desc["scols"]:
                                    vals[e] = bufs[1][eoff(1, off[1], e)]
                        for e in range(V):
                            bufs[0][eoff(0, off[0], e)] = vals[e]
                    elif op == "dot":
                        for e in range(V):
                            slots[0] += float(bufs[0][eoff(0, off[0], e)]) * \
                                float(bufs[1][eoff(1, off[1], e)])
                    elif op == "update":
                        for e in range(V):
                            xi = eoff(0, off[0], e)
                            x, y, z = bufs[0][xi], bufs[1][eoff(1, off[1], e)], bufs[2][eoff(2, off[2], e)]
                            bufs[0][xi] = (x + (y * x)) - z
                    elif op == "binary":
                        fn = {"add": np.add, "sub": np.subtract, "mul": np.multiply,
                              "div": np.divide}[binop]
                        for e in range(V):
                            with np.errstate(all="ignore"):
                                bufs[0][eoff(0, off[0], e)] = fn(bufs[1][eoff(1, off[1], e)],
                                                                 bufs[2][eoff(2, off[2], e)])
                    else:
                        x = [float(bufs[0][eoff(0, off[0], e)]) for e in range(V)]
                        s_ = sum(x)
                        for k in range(D - 1):
                            slots[k] += u[k] * s_
                        wr = sum((e >> lgL) * x[e] for e in range(V))
                        wc = sum((e & (L - 1)) * x[e] for e in range(V))
                        base = uv * (desc["rowmul"] + desc["colmul"])
                        if desc["collapsed"]:
                            slots[D - 1] += base * s_ + wr
                            slots[D] += wc
                        else:
                            slots[D - 1] += base * s_ + wc
                u, off, oob = step(u, off, oob)
                v += dv
    if op == "dot":
        return slots[0]
    if op == "ev":
        d = desc["d"]
        return [slots[sl] if sl >= 0 else 0.0 for sl in desc["slot_of_axis"][:d]]
    return None


def run_flat(desc: dict, op: str, bufs: list, binop: str = "mul"):
    """Flat vectors: vector v is counter elements [v*V, v*V+V); the lane walks them with the
    +1 odometer (Alg 3), then skips (dv-1)*V elements with the mixed-radix step."""
    D, V, idx64 = desc["D"], desc["V"], desc["idx64"]
    ext, dlt, bnd = desc["ext"], desc["dlt"], desc["bnd"]
    khi, klo = desc["khi"], desc["klo"]
    T = desc["t"]
    nt = len(T)
    N, nvec = desc["N"], desc["nvec"]
    W = lambda x: _wrap(x, idx64)
    slots = [0.0] * (D + 2)

    def start(f):
        u = [0] * D
        for k in range(D - 1, 0, -1):
            u[k] = f % ext[k]
            f //= ext[k]
        u[0] = f
        off = [W(sum(u[k] * T[x]["sig"][k] for k in range(D))) for x in range(nt)]
        return u, off

    def inc1(u, off):
        off = [W(off[x] + T[x]["sig"][D - 1]) for x in range(nt)]
        for k in range(D - 1, -1, -1):
            nu = u[k] + 1
            carry = k > 0 and nu >= ext[k]
            if carry:
                nu = 0
                off = [W(off[x] + T[x]["kap"][k]) for x in range(nt)]
            u[k] = nu
            if not carry:
                break
        return u, off

    def skip(u, off):
        off = [W(off[x] + T[x]["step"]) for x in range(nt)]
        carry = 0
        for k in range(D - 1, -1, -1):
            if k > khi:
                continue
            nu = u[k] + dlt[k] + carry
            carry = int(nu >= ext[k])
            if carry:
                nu -= ext[k]
                off = [W(off[x] + T[x]["kap"][k]) for x in range(nt)]
            u[k] = nu
            if k <= klo and not carry:
                break
        return u, off

    wmul, wspan, dv = desc["wmul"], desc["wspan"], desc["dv"]
    units = (nvec + wmul - 1) // wmul if desc["mode"] == 0 else dv // 32
    fn = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide}.get(binop)
    for w in range(units):
        base0 = w * wmul
        if base0 >= nvec:
            continue
        vend = min(base0 + wspan, nvec)
        for lane in range(32):
            v = base0 + lane
            u, off = start(v * V)
            while v < vend:
                for e in range(V):
                    f = v * V + e
                    if f < N:
                        if op == "embed":
                            inb = all(u[k] < bnd[k] for k in range(D))
                            bufs[0][off[0]] = bufs[1][off[1]] if inb else 0
                        elif op == "binary":
                            with np.errstate(all="ignore"):
                                bufs[0][off[0]] = fn(bufs[1][off[1]], bufs[2][off[2]])
                        elif op == "ev":
                            x = float(bufs[0][off[0]])
                            for k in range(D):
                                slots[k] += u[k] * x
                    u, off = inc1(u, off)
                u, off = skip(u, off)
                v += dv
    if op == "ev":
        d = desc["d"]
        return [slots[sl] if sl >= 0 else 0.0 for sl in desc["slot_of_axis"][:d]]
    return None


def run_rows(desc: dict, op: str, bufs: list, binop: str = "mul"):
    """Row windows: lane i of warp step s holds counter row 32s+i (its tensor offsets and embed
    bound, kept by the odometer); the warp sweeps the window's 32*n elements, element
    e = 32j + lane in row umulhi(e, rmag) (== e // n, checked), column e - row*n, reading the
    row's rebased offsets from the warp's row table as the kernel does."""
    D, idx64 = desc["D"], desc["idx64"]
    ext, dlt, bnd = desc["ext"], desc["dlt"], desc["bnd"]
    khi, klo = desc["khi"], desc["klo"]
    T = desc["t"]
    nt = len(T)
    n, mg, m = desc["rowlen"], desc["rmag"], desc["scols"]
    nvec = desc["nvec"]
    W = lambda x: _wrap(x, idx64)
    fn = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide}.get(binop)

    def start(v):
        u = [0] * D
        for k in range(D - 1, 0, -1):
            u[k] = v % ext[k]
            v //= ext[k]
        u[0] = v
        off = [W(sum(u[k] * T[x]["sig"][k] for k in range(D))) for x in range(nt)]
        oob = any(u[k] >= bnd[k] for k in range(D))
        return u, off, oob

    def step(u, off):
        off = [W(off[x] + T[x]["step"]) for x in range(nt)]
        carry = 0
        for k in range(D - 1, -1, -1):
            if k > khi:
                continue
            nu = u[k] + dlt[k] + carry
            carry = int(nu >= ext[k])
            if carry:
                nu -= ext[k]
                off = [W(off[x] + T[x]["kap"][k]) for x in range(nt)]
            u[k] = nu
            if k <= klo and not carry:
                break
        return u, off, any(u[k] >= bnd[k] for k in range(D))

    wmul, wspan, dv = desc["wmul"], desc["wspan"], desc["dv"]
    units = (nvec + wmul - 1) // wmul if desc["mode"] == 0 else dv // 32
    Wg = desc["rwin"] if dv == 32 else 1
    K = 32 // desc["esz"]
    for w in range(units):
        base0 = w * wmul
        if base0 >= nvec:
            continue
        vend = min(base0 + wspan, nvec)
        lanes = [start(base0 + i) for i in range(32)]
        b = base0
        while b < vend:
            # the warp's row table: Wg windows of 32 rows (fewer at the end of its range); each
            # entry holds the tensors' offsets rebased to the group's element index
            # (off - r0*tau, r0 = the row's first element) and, for embed, the bound r0 + m
            gb = b * n
            tab, rows, wi = [], 0, 0
            while wi < Wg and b < vend:
                nr = min(32, vend - b)
                for i in range(32):
                    u, off, oob = lanes[i]
                    r0 = (32 * wi + i) * n
                    ent = [W(off[x] - r0 * T[x]["tau"]) for x in range(nt)]
                    mr = m
                    if desc.get("seglen"):   # a segment of a split axis: per-segment bound
                        mr = max(0, min(desc["segm"] - u[D - 1] * n, n))
                    lim = r0 + mr if (i < nr and not oob) else 0
                    tab.append((ent, lim))
                rows = 32 * wi + nr
                lanes = [step(list(u), off) for (u, off, _) in lanes]
                b += dv
                wi += 1
            tot = rows * n
            for e in range(0, (tot + 32 * K - 1) // (32 * K) * 32 * K):
                row = (e * mg) >> 32
                assert row == e // n, (e, n, mg)
                if e >= tot:
                    continue
                ent, lim = tab[row]
                o = [W(ent[x] + e * T[x]["tau"]) for x in range(nt)]
                if T[0]["vec"]:
                    assert o[0] == gb + e
                if op == "embed":
                    bufs[0][o[0]] = bufs[1][o[1]] if e < lim else 0
                else:
                    with np.errstate(all="ignore"):
                        bufs[0][o[0]] = fn(bufs[1][o[1]], bufs[2][o[2]])
    return None
