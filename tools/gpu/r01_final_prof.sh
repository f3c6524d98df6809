set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_step -s 12 -c 2 -o gpurun_out/prof_bench_step python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>&1; echo "step prof rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_tc -s 4 -c 2 -o gpurun_out/prof_dense_tc python tools/large_bench.py 4096 > /dev/null 2>&1; echo "dense prof rc=$?"
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=3, packed=False)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe_matvec -s 1 -c 1 -o gpurun_out/prof_pipe_scale python /tmp/one.py > /dev/null 2>&1; echo "pipe prof rc=$?"
