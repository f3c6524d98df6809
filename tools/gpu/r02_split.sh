for v in split8; do QMOE_LIB_PATH=variants/$v/libqmoe.so python -m pytest tests -m gpu -q -x -k "fused or moe or model or step" 2>&1 | tail -1; done
for l in product variants/split1/libqmoe.so variants/split2/libqmoe.so variants/split4/libqmoe.so variants/split8/libqmoe.so; do
  export QMOE_LIB_PATH=$l; [ $l = product ] && unset QMOE_LIB_PATH
  python tools/moe_sweep.py 1 2 4 8 16 2>&1; WORKLOAD=switch-c2048 python tools/moe_sweep.py 1 8 2>&1
done
