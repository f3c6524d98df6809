set -x
cat > /tmp/one.py <<'PY'
import sys; sys.argv=['x']
sys.path.insert(0,'tools')
import seg_bench as S
S.bench(768, 3072, ntok=1, iters=3)
S.bench(3072, 768, ntok=1, iters=3)
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_matvec -s 1 -c 1 -o gpurun_out/prof_seg_wo python /tmp/one.py > gpurun_out/prof_seg.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_matvec -s 5 -c 1 -o gpurun_out/prof_seg_wi python /tmp/one.py > gpurun_out/prof_seg2.log 2>&1; echo "ncu rc=$?"
