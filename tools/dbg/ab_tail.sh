# A/B of the reduction tail on one box (C3, B2): per-block timelines of the current sources,
# then cold ncu launch times and back-to-back graph times of the current build (cur) and of
# tools/dbg/libs/libtriot_<v>.so for each v in "$@" (e.g. base = the previous commit's build).
set -u
O=gpurun_out
for what in --ldg --dot; do
  echo "== probe $what" >> $O/tail_probe.log
  python tools/ev_probe.py $what >> $O/tail_probe.log 2>&1
done
for rep in 1 2; do
for v in cur "$@"; do
  L=""
  [ $v != cur ] && L=tools/dbg/libs/libtriot_$v.so
  echo "== b2b $v rep $rep" >> $O/tail_b2b.log
  TRIOT_LIB_PATH=$L python tools/dbg/b2b.py >> $O/tail_b2b.log 2>&1
  TRIOT_LIB_PATH=$L python tools/profile_ops.py --only C3,B2 --reps 5 > /dev/null 2>&1 && \
  TRIOT_LIB_PATH=$L ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv \
     --log-file $O/tail_ncu_${v}_$rep.csv python tools/profile_ops.py --only C3,B2 --reps 5 > /dev/null 2>&1
done
done
python tools/dbg/ncu_times.py $O/tail_ncu_*.csv > $O/tail_ncu_summary.txt 2>&1
cat $O/tail_ncu_summary.txt
cat $O/tail_b2b.log
