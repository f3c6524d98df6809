python -m pytest tests -m gpu -q -x -k "fused_step or plan or fullshape or model or hash or moe_tiny or routed or ep" > gpurun_out/iter_tests.log 2>&1; tail -2 gpurun_out/iter_tests.log
python tools/step_trace.py 1 64 2>&1 | grep "^T="
python tools/debug/plan_cost.py 2>&1
python tools/moe_sweep.py 1 8 32 64 128 160 256 2>&1
WORKLOAD=switch-c2048 python tools/moe_sweep.py 1 64 256 2>&1
