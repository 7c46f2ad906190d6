# usage: bash tools/dbg/ab_lib.sh OPS VARIANT  -- cold ncu launch times, current build vs
# tools/dbg/libs/libtriot_VARIANT.so, same box (after a plain run of each)
OPS=$1; V=$2
python tools/profile_ops.py --only $OPS --reps 5 > /dev/null
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_$V.so python tools/profile_ops.py --only $OPS --reps 5 > /dev/null
ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file gpurun_out/ab_base.csv python tools/profile_ops.py --only $OPS --reps 5 > /dev/null 2>&1
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_$V.so ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file gpurun_out/ab_$V.csv python tools/profile_ops.py --only $OPS --reps 5 > /dev/null 2>&1
