timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
QMOE_LAYOUT=raw timeout 300 python tools/moe_sweep.py -1 1 8 64 256
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_matvec -s 40 -c 2 -o gpurun_out/prof_moe64 python tools/moe_sweep.py -1 64 > gpurun_out/prof_moe64.log 2>&1; echo "ncu rc=$?"
