ncu --set full --import-source on --clock-control none -k regex:moe_step_kernel --launch-skip 25 -c 1 -o gpurun_out/t1_step -f python tools/debug/t1_chain.py > gpurun_out/t1prof.log 2>&1
T=64 ncu --set full --import-source on --clock-control none -k regex:moe_step_kernel --launch-skip 25 -c 1 -o gpurun_out/t64_step -f python tools/debug/t1_chain.py >> gpurun_out/t1prof.log 2>&1
tail -3 gpurun_out/t1prof.log
