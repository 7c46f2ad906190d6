# row-window zoo + views: the current build vs tools/dbg/libs/libtriot_prev.so, same box
python tools/shape_zoo.py --rows | sed 's/^{/{"lib": "new", /'
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so python tools/shape_zoo.py --rows | sed 's/^{/{"lib": "prev", /'
python tools/shape_zoo.py --views | sed 's/^{/{"lib": "new", /'
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so python tools/shape_zoo.py --views | sed 's/^{/{"lib": "prev", /'
