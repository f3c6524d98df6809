# GPU suite + both bench arms (default flags, as the driver runs them)
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_iter.log 2>&1; tail -3 gpurun_out/pytest_gpu_iter.log
timeout 900 python bench.py > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench_iter.log | cut -c1-3000
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_iter.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_iter.log | cut -c1-400
