timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r01.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r01.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r01.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_r01.log
timeout 300 python tools/moe_sweep.py -1 1 8 64 256
