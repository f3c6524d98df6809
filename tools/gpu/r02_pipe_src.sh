# ncu source-level (SASS) instruction counts of the at-scale streaming kernel
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=3, packed=False)
PY
timeout 900 ncu --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:pipe_matvec -s 1 -c 1 -o gpurun_out/pipe_src python /tmp/one.py > gpurun_out/pipe_src.log 2>&1; echo "rc=$?"
for lg in 0 1 2 3; do
cat > /tmp/lg.py <<PY
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=$lg, ntok=1, iters=10, packed=False)
S.bench(3072, 768, lg=$lg, ntok=1, iters=10, packed=False)
PY
timeout 300 python /tmp/lg.py >> gpurun_out/lg_sweep.log 2>&1
done
