# Round-2 start: GPU suite, bench, and the at-scale kernel counters that the
# instruction-per-codeword work is judged on.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02a.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02a.log
timeout 900 python bench.py > gpurun_out/bench_r02a.log 2>&1; tail -1 gpurun_out/bench_r02a.log | cut -c1-400
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=3, packed=False)
PY
timeout 600 ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pipe_matvec -s 1 -c 1 --csv python /tmp/one.py > gpurun_out/pipe_counters_r02a.csv 2>&1; echo "pipe rc=$?"
