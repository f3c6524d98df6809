set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02b.log 2>&1; tail -1 gpurun_out/pytest_gpu_r02b.log
timeout 900 python bench.py > gpurun_out/bench_r02b.log 2>&1; echo "bench rc=$?"
LAYERS=30 timeout 1500 python tools/c2048_model.py 1 8 64 > gpurun_out/c2048_model_r02.jsonl 2>&1; echo "model rc=$?"
