# A/B: product build vs variants/$1 (step sweeps + at-scale kernel)
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=10)
S.bench(3072, 768, lg=0, ntok=1, iters=10)
S.bench(768, 3072, lg=2, ntok=2, iters=10)
PY
for l in product variants/$1/libqmoe.so; do
  export QMOE_LIB_PATH=$l; [ $l = product ] && unset QMOE_LIB_PATH
  echo "== $l"
  python tools/moe_sweep.py 1 8 64 128 2>&1
  WORKLOAD=switch-c2048 python tools/moe_sweep.py 1 64 2>&1
  timeout 600 python /tmp/one.py 2>&1 | tail -3
done
