# A/B of experiment builds (variants/*/libqmoe.so): fused step T=1/8/64 and the kernel at scale
cat > /tmp/seg.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=10)
S.bench(3072, 768, lg=0, ntok=1, iters=10)
PY
for v in ${VARIANTS:-v0 v1 v2 v3}; do
  QMOE_LIB_PATH=variants/$v/libqmoe.so timeout 300 python tools/moe_sweep.py 1 8 64 2>&1 | grep step
  QMOE_LIB_PATH=variants/$v/libqmoe.so timeout 300 python /tmp/seg.py 2>&1 | grep raw | sed "s/^/$v /"
done
