python -m pytest tests -m gpu -q -x -k "fused_step or plan or fullshape or model or hash or moe_tiny or routed" > gpurun_out/quad_tests.log 2>&1; tail -3 gpurun_out/quad_tests.log
for lib in product variants/oldplan/libqmoe.so; do
  if [ $lib = product ]; then unset QMOE_LIB_PATH; else export QMOE_LIB_PATH=$lib; fi
  echo "== $lib"
  python tools/debug/plan_cost.py 2>&1
  python tools/moe_sweep.py 1 8 64 128 160 256 2>&1
  WORKLOAD=switch-c2048 python tools/moe_sweep.py 1 64 256 2>&1
done
