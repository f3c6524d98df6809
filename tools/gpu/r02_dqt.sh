for v in $VARIANTS; do
  echo "== $v"
  QMOE_LIB_PATH=variants/$v/libqmoe.so timeout 600 python tools/large_bench.py ${TS:-1024 4096} 2>&1 | grep "^{\|Error" | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(d['T'], d['step_us']['dense'])
    except Exception: print(l[:200])"
done
