for i in 1 2; do
python tools/shape_zoo.py --rows | sed "s/^{/{\"lib\": \"rows$i\", /"
TRIOT_LIB_PATH=tools/dbg/libs/libtriot_prev.so python tools/shape_zoo.py --rows | sed "s/^{/{\"lib\": \"prev$i\", /"
done
