timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_fullshape.py -q -x -k "dense" 2>&1 | tail -3
for l in product variants/densrw/libqmoe.so; do
  export QMOE_LIB_PATH=$l; [ $l = product ] && unset QMOE_LIB_PATH
  echo "== $l"
  timeout 600 python tools/large_bench.py 1024 4096 2>&1 | grep "^{" | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['T'], d['step_us'])"
done
