# Build tools/dbg/libs/libtriot_<name>.so with capi + the EV (f64) and inner-product (f64)
# families recompiled with extra defines (A/B of reduction layout constants that the host side
# must agree on, e.g. -DTRIOT_EV_MINPAD=4).
#   bash tools/dbg/build_variant3.sh <name> "<defines>"
set -e
NAME=$1; DEFS=$2
B=paper_1608_00099_b200/build; C=paper_1608_00099_b200/csrc
OUT=tools/dbg/libs/build_$NAME; mkdir -p $OUT tools/dbg/libs
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fvisibility=hidden -I $C -I include -diag-suppress 177 --compress-mode=size"
nvcc $FLAGS $DEFS -DTRIOT_INST_OP=2 -DTRIOT_INST_ESZ=8 -c $C/inst.cu -o $OUT/inst_2_8_0.o &
nvcc $FLAGS $DEFS -DTRIOT_INST_OP=3 -DTRIOT_INST_ESZ=8 -c $C/inst.cu -o $OUT/inst_3_8_0.o &
nvcc $FLAGS $DEFS -c $C/capi.cu -o $OUT/capi.o &
wait
OBJS=""
for o in $B/*.o; do b=$(basename $o); if [ -f $OUT/$b ]; then OBJS="$OBJS $OUT/$b"; else OBJS="$OBJS $o"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/dbg/libs/libtriot_$NAME.so $OBJS -Xcompiler -fvisibility=hidden -Xlinker --exclude-libs,ALL
ls -la tools/dbg/libs/libtriot_$NAME.so
