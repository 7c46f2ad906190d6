# Row windows vs flat vectors on the short-odd-row and misaligned-output zoo, same box
# (tools/dbg/ab_table.py prints the comparison); with tools/dbg/libs/libtriot_prev.so present,
# also the previous build of the row-window kernels.
python tools/shape_zoo.py --rows | sed 's/^{/{"lib": "rows", /'
python tools/shape_zoo.py --rows --policy 5,0 | sed 's/^{/{"lib": "flat", /'
if [ -f tools/dbg/libs/libtriot_prev.so ]; then
  TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so python tools/shape_zoo.py --rows | sed 's/^{/{"lib": "prev", /'
fi
