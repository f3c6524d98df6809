# Round-1 end-of-round evidence: tests, smoke, bench (both arms), launch list,
# ncu captures of the fused step, the dense pass and the kernel at scale.
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_end.log 2>&1; tail -1 gpurun_out/pytest_gpu_end.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_end.log 2>&1; tail -1 gpurun_out/smoke_end.log
timeout 900 python bench.py > gpurun_out/bench_end.log 2>&1; tail -1 gpurun_out/bench_end.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_end.log 2>&1; tail -1 gpurun_out/bench_ref_end.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_end.csv python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_step -s 12 -c 2 -o gpurun_out/prof_step_end python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>&1; echo "step prof rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_rw -s 4 -c 2 -o gpurun_out/prof_dense_end python tools/large_bench.py 4096 > /dev/null 2>&1; echo "dense prof rc=$?"
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=3, packed=False)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe_matvec -s 1 -c 1 -o gpurun_out/prof_pipe_end python /tmp/one.py > /dev/null 2>&1; echo "pipe prof rc=$?"
timeout 300 python tools/router_bench.py > gpurun_out/router_end.log 2>&1
timeout 300 python tools/e2e_breakdown.py 64 > gpurun_out/e2e_end.log 2>&1
timeout 600 python tools/moe_sweep.py -1 1 8 64 256 > gpurun_out/sweep_end.log 2>&1
timeout 900 python tools/large_bench.py 1024 4096 > gpurun_out/large_end.log 2>&1
WORKLOAD=switch-base-128 timeout 600 python tools/large_bench.py 2048 >> gpurun_out/large_end.log 2>&1
timeout 600 python tools/step_trace.py 1 8 64 256 > gpurun_out/trace_end.log 2>&1
