# A/B of the config ops on one box: the current build vs tools/dbg/libs/libtriot_prev.so
# (cold-cache ncu launch times, 5 launches each, after a plain run of each).
python tools/profile_ops.py --only C2,C3,C4,C5,B2,B3 --reps 5 > /dev/null
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so python tools/profile_ops.py --only C2,C3,C4,C5,B2,B3 --reps 5 > /dev/null
ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file gpurun_out/ab_ops_new.csv python tools/profile_ops.py --only C2,C3,C4,C5,B2,B3 --reps 5 > /dev/null 2>&1
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file gpurun_out/ab_ops_prev.csv python tools/profile_ops.py --only C2,C3,C4,C5,B2,B3 --reps 5 > /dev/null 2>&1
