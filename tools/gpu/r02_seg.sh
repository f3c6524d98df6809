# at-scale kernel throughput for the main shapes (+ optional ncu counters)
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=10)
S.bench(768, 3072, lg=1, ntok=1, iters=10)
S.bench(3072, 768, lg=0, ntok=1, iters=10)
S.bench(3072, 768, lg=1, ntok=1, iters=10)
S.bench(768, 3072, lg=2, ntok=2, iters=10)
PY
timeout 600 python /tmp/one.py > gpurun_out/seg_iter.log 2>&1; cat gpurun_out/seg_iter.log
cat > /tmp/two.py <<'PY'
import sys; sys.path.insert(0, 'tools')
import seg_bench as S
S.bench(768, 3072, lg=2, ntok=1, iters=3)
PY
timeout 600 ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pipe_matvec -s 1 -c 1 --csv python /tmp/two.py > gpurun_out/pipe_counters_iter.csv 2>&1
grep -v "^==" gpurun_out/pipe_counters_iter.csv | grep pipe_matvec | awk -F'","' '{print $(NF-2), $NF}'
