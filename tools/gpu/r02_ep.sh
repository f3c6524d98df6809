# EP path on one GPU (torchrun world 1 through the expert-parallel code path), c2048-shaped layer
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --force-ep --workload switch-c2048 --steps 10 --warmup 3 > gpurun_out/ep_c2048.log 2>&1; echo "ep rc=$?"; tail -2 gpurun_out/ep_c2048.log | cut -c1-1500
