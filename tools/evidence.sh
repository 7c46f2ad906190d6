# Round evidence (run on a B200 through gpurun from the repo root; writes gpurun_out/):
#   bench line, reference arm, ncu launch list of the bench command, and one ncu --set full
#   capture of the step kernels, the row-window kernels and Benchmarks 2-4, summarised into
#   JSON on the box (the .ncu-rep itself stays in /tmp: it exceeds gpurun's copy-back limit),
#   and profiles/traffic.json regenerated from it (bench.py's roofline.traffic source).
#   ROUND=r02 bash tools/evidence.sh
set -u
R=${ROUND:-rXX}
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-isolated --e2e-steps 1 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/${R}_launches_bench.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-isolated --e2e-steps 1 > /dev/null 2>&1
OPS=C2,C3,C4,C5,ROWS7,ROWSB63,B2,B3,B4
python tools/profile_ops.py --only $OPS --reps 1 > /dev/null && \
  ncu --set full --import-source on --cache-control all --clock-control none \
      --metrics smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio,smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      -k regex:"embed|binary|ev_kernel|dot_kernel|update_kernel|conv_kernel" -o /tmp/prof_ops \
      python tools/profile_ops.py --only $OPS --reps 1 > gpurun_out/${R}_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof_ops.ncu-rep --json gpurun_out/${R}_ncu_full_ops.json > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_ops.ncu-rep --evidence C2,C3,C4,C5 --json gpurun_out/${R}_ncu_evidence.json > /dev/null 2>&1
python tools/traffic_from_ncu.py gpurun_out/${R}_ncu_full_ops.json $OPS $R > gpurun_out/${R}_traffic.json
ls -la gpurun_out
