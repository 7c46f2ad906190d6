# EV / inner product / update launch-policy sweep under ncu (cold-cache launch times per policy)
set -e
POLS="-1,0 4,4 4,8 4,16 4,32 0,8 0,16"
for p in $POLS; do python tools/profile_ops.py --only C3,B2,B3 --reps 5 --policy=$p > /dev/null; done
for p in $POLS; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control all --clock-control none --csv --log-file gpurun_out/ncu_ev_pol_${p}.csv python tools/profile_ops.py --only C3,B2,B3 --reps 5 --policy=$p > /dev/null
done
