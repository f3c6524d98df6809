set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi2.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 4 --warmup 3 > gpurun_out/launches_run.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lean_matvec -s 20 -c 2 -o gpurun_out/prof_lean python bench.py --profile --steps 4 --warmup 3 > gpurun_out/prof_run.log 2>&1; echo "ncu2 rc=$?"
tail -c 2500 gpurun_out/bench.log
