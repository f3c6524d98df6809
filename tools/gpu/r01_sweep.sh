timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/seg_bench.py 2>&1 | head -4
for H in 2048 8192 16384 32768 -1; do timeout 300 python tools/moe_sweep.py $H 1 8 64 256; done
