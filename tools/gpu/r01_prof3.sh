timeout 600 python tools/seg_bench.py 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe_matvec -s 40 -c 2 -o gpurun_out/prof_pipe64 python tools/moe_sweep.py -1 64 > gpurun_out/prof_pipe64.log 2>&1; echo "ncu rc=$?"
