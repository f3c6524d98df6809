K="test_fused_step_equals_grouped_passes_and_plan or test_moe_tiny or test_moe_dense_decode_then_mma_vs_oracle or test_worked_examples or test_long_rows or test_host_forward_graph or test_routed_gated or test_hash_rule or test_argmax_rule or test_ep_slots or test_fused_plan_many or test_read_checkpoint_device or test_load_moe_layer"
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/san_$tool.log | tail -4
done
