"""Multi-process (gloo, world size 2, CPU) tests of the slab-sharding host logic
(paper_1608_00099_b200/parallel.py): slab bounds cover every row once, the per-rank embed and
binary slabs tile the global result with no collective, and the sharded expected value -- with
the oracle standing in for each rank's GPU kernel -- equals the oracle on the whole tensor."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1608_00099_b200 import parallel as P
from triot_inputs import make_inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_ev_offset(p_slab, offset):
    """Stand-in for triot_expected_value_offset: the oracle's sums, each weight shifted by the
    slab's origin (sum_t (off_k + t_k) p[t] = m_k + off_k * mass)."""
    p = p_slab.numpy()
    m = O.expected_value(p)
    mass = float(np.sum(p, dtype=np.float64))
    return torch.tensor([m[k] + offset[k] * mass for k in range(p.ndim)], dtype=torch.float64)


def _rank_order_sum(rows):
    """Stand-in for triot_sum_rows: rows added in order."""
    out = torch.zeros(rows.shape[1], dtype=torch.float64)
    for r in range(rows.shape[0]):
        out += rows[r]
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        # expected value over a slab of C3's axis 0 (integer-valued copy: exact) and C3 itself
        p_int = np.random.default_rng(5).integers(0, 256, size=(7, 5, 6, 3)).astype(np.float64)
        p_c3 = make_inputs("C3")["p"][:, :4, :4].copy()
        for name, p in (("int", p_int), ("c3", p_c3)):
            lo, hi = P.slab_rows(p.shape[0], world, rank)
            got = P.expected_value_sharded(torch.from_numpy(p[lo:hi].copy()), lo,
                                           local_ev=_oracle_ev_offset, sum_rows=_rank_order_sum)
            res[name] = got.numpy()
        # embed slab: each rank's slab of dst from the global src, oracle as the local kernel
        src = make_inputs("C1")["src"]
        dst_shape = (8, 16, 8, 8)
        lo, hi = P.slab_rows(dst_shape[0], world, rank)
        slab = np.empty((hi - lo,) + dst_shape[1:])
        O.embed(slab, src[lo:min(hi, src.shape[0])].copy())
        res["embed"] = (lo, hi, slab)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_ev_and_slabs_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    p_int = np.random.default_rng(5).integers(0, 256, size=(7, 5, 6, 3)).astype(np.float64)
    ref_int = O.expected_value(p_int)
    p_c3 = make_inputs("C3")["p"][:, :4, :4].copy()
    ref_c3 = O.expected_value(p_c3)
    for r in range(world):
        np.testing.assert_array_equal(out[r]["int"], ref_int)          # exact
        assert np.all(np.abs(out[r]["c3"] - ref_c3) <= 1e-12 * np.abs(ref_c3))
    assert np.array_equal(out[0]["c3"], out[1]["c3"])                  # same on every rank
    # embed slabs tile the global result
    full = np.empty((8, 16, 8, 8))
    O.embed(full, make_inputs("C1")["src"])
    rows = []
    for r in range(world):
        lo, hi, slab = out[r]["embed"]
        rows.append((lo, hi))
        np.testing.assert_array_equal(slab, full[lo:hi])
    assert sorted(rows)[0][0] == 0 and sorted(rows)[-1][1] == 8


def test_slab_rows_cover_once():
    for n0 in (0, 1, 5, 16, 384, 511):
        for world in (1, 2, 3, 8):
            spans = [P.slab_rows(n0, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n0
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_leading_box_partition_covers_once():
    """Every element of the shape lies in exactly one rank's box (C2/C3/C4/C5 shapes at 1..8
    ranks, including (4,)*14 with more ranks than axis-0 indices)."""
    for shape in [(512, 512, 512), (16,) * 6, (32, 32, 24, 32, 32), (4,) * 14, (3, 5), (2, 2, 2),
                  (1, 7), (5,)]:
        for world in range(1, 9):
            lead = shape[:3]
            cover = np.zeros(lead, dtype=np.int32)
            for r in range(world):
                box = P.leading_box(shape, world, r)
                assert all(0 <= lo <= hi <= n for (lo, hi), n in zip(box, shape))
                assert all(box[k] == (0, shape[k]) for k in range(3, len(shape)))
                cover[tuple(slice(lo, hi) for lo, hi in box[:3])] += 1
            assert np.all(cover == 1), (shape, world)


def test_bench_slab_plan_reassembles_the_global_step():
    """bench.slab_plan at 1..8 ranks: every rank's blocks, run through the oracle, reassemble the
    global C2/C4/C5 outputs exactly, and the rank results of C3 (offset EVs, rank-order sum)
    equal the global oracle EV -- on shrunken copies of the configs (same dimensions, smaller
    extents) so the oracle finishes fast."""
    import bench
    rng = np.random.default_rng(11)
    host = {
        "C2": {"src": rng.standard_normal((6, 5, 7)).astype(np.float32), "dst_shape": (9, 8, 8)},
        "C3": {"p": rng.random((5, 4, 3, 4))},
        "C4": {"a": rng.random((4, 6, 3, 5)), "b": rng.random((6, 4, 4, 4)),
               "iter_shape": (4, 4, 3, 4)},
        "C5": {"src": rng.random((3,) * 6).astype(np.float32), "dst_shape": (4,) * 6},
    }
    ref2 = np.empty(host["C2"]["dst_shape"], np.float32); O.embed(ref2, host["C2"]["src"])
    ref5 = np.empty(host["C5"]["dst_shape"], np.float32); O.embed(ref5, host["C5"]["src"])
    ref4 = O.apply_binary(host["C4"]["a"], host["C4"]["b"], "mul", iter_shape=(4, 4, 3, 4))
    ref3 = O.expected_value(host["C3"]["p"])
    for world in range(1, 9):
        out2 = np.full(ref2.shape, np.nan, np.float32)
        out5 = np.full(ref5.shape, np.nan, np.float32)
        out4 = np.full(ref4.shape, np.nan)
        tot3 = np.zeros(4)
        for r in range(world):
            sl = bench.slab_plan(host, world, r)
            for n, out in (("C2", out2), ("C5", out5)):
                blk = np.empty(sl[n]["dst_shape"], np.float32)
                if blk.size:
                    O.embed(blk, sl[n]["src"])
                out[tuple(slice(lo, hi) for lo, hi in sl[n]["box"])] = blk
            if all(e > 0 for e in sl["C4"]["iter_shape"]):
                blk = O.apply_binary(sl["C4"]["a"], sl["C4"]["b"], "mul",
                                     iter_shape=sl["C4"]["iter_shape"])
                out4[tuple(slice(lo, hi) for lo, hi in sl["C4"]["box"])] = blk
            p = sl["C3"]["p"]
            if p.size:
                m, mass = O.expected_value(p), p.sum()
                tot3 = tot3 + np.array([m[k] + sl["C3"]["offset"][k] * mass for k in range(4)])
        np.testing.assert_array_equal(out2, ref2)
        np.testing.assert_array_equal(out5, ref5)
        np.testing.assert_array_equal(out4, ref4)
        assert np.all(np.abs(tot3 - ref3) <= 1e-12 * np.abs(ref3)), world
