# Round-2 evidence: tests, smoke, bench (both arms), launch list, ncu captures
# (fused step, kernel at scale, dense pass), sweeps, traces, reference tests,
# sanitizers.
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02.log 2>&1; tail -1 gpurun_out/pytest_gpu_r02.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; tail -1 gpurun_out/smoke_r02.log
timeout 900 python bench.py > gpurun_out/bench_r02.log 2>&1; tail -1 gpurun_out/bench_r02.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r02.log 2>&1; tail -1 gpurun_out/bench_ref_r02.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:moe_step -s 12 -c 2 -o gpurun_out/prof_step_r02 python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>&1; echo "step prof rc=$?"
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=3)
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_matvec -s 1 -c 1 -o gpurun_out/prof_pipe_r02 python /tmp/one.py > /dev/null 2>&1; echo "pipe prof rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_ -s 30 -c 2 -o gpurun_out/prof_dense_r02 python tools/large_bench.py 4096 > /dev/null 2>&1; echo "dense prof rc=$?"
timeout 600 python tools/moe_sweep.py 1 2 4 8 16 32 64 128 160 256 > gpurun_out/sweep_r02.log 2>&1
WORKLOAD=switch-c2048 timeout 900 python tools/moe_sweep.py 1 8 64 256 > gpurun_out/sweep_c2048_r02.log 2>&1
timeout 600 python tools/step_trace.py 1 8 64 256 > gpurun_out/trace_r02.log 2>&1
timeout 900 python tools/large_bench.py 512 768 1024 4096 > gpurun_out/large_r02.log 2>&1
WORKLOAD=switch-base-128 timeout 900 python tools/large_bench.py 1024 2048 > gpurun_out/large_base_r02.log 2>&1
cat > /tmp/seg.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
for rows, cols, lg in ((3072, 768, 0), (768, 3072, 2), (6144, 2080, 1), (2080, 6144, 2)):
    for ntok in (1, 2):
        S.bench(rows, cols, lg=lg, ntok=ntok, iters=10)
PY
timeout 900 python /tmp/seg.py > gpurun_out/seg_r02.log 2>&1
tools/reference_tests.sh run > gpurun_out/reference_tests_r02.txt 2>&1
bash tools/gpu/sanitize.sh > gpurun_out/sanitize_r02.log 2>&1; tail -12 gpurun_out/sanitize_r02.log
