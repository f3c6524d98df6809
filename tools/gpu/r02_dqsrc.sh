export QMOE_LIB_PATH=variants/${V:-dq_r2b3}/libqmoe.so
timeout 900 ncu --section WarpStateStats --section SourceCounters --section InstructionStats --import-source on --clock-control none -k regex:dense_dq --launch-skip 30 -c 1 -o gpurun_out/dq_src -f python tools/large_bench.py 4096 > gpurun_out/dq_src.log 2>&1
tail -3 gpurun_out/dq_src.log
