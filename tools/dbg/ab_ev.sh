# A/B of the expected value / inner product on one box: the current build vs tools/dbg/libs/
# libtriot_prev.so, cold-cache ncu launch times (5 each).
python tools/profile_ops.py --only C3,B2 --reps 5 > /dev/null
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so python tools/profile_ops.py --only C3,B2 --reps 5 > /dev/null
ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file gpurun_out/ab_ev_new.csv python tools/profile_ops.py --only C3,B2 --reps 5 > /dev/null 2>&1
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file gpurun_out/ab_ev_prev.csv python tools/profile_ops.py --only C3,B2 --reps 5 > /dev/null 2>&1
