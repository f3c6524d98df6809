#!/bin/bash
# Re-run the reference's own test modules against the drop-in.
#   stage (here, where /root/reference exists):  tools/reference_tests.sh stage
#     copies /root/reference/pkg/tests into baseline/_ref/tests (git-ignored,
#     travels to the GPU box with the snapshot; never committed)
#   run (on the GPU box):                        tools/reference_tests.sh run
#     `import moepack` -> tools/ref_shim (this repo's package), one pytest per module
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "${1:-run}" = stage ]; then
  rm -rf "$ROOT/baseline/_ref/tests" && mkdir -p "$ROOT/baseline/_ref" && cp -r /root/reference/pkg/tests "$ROOT/baseline/_ref/tests"
  echo "staged $(ls "$ROOT/baseline/_ref/tests" | wc -l) files"
  exit 0
fi
cd "$ROOT/baseline/_ref/tests" || exit 1
for m in test_bf16 test_dictionary test_codec test_stats test_cli test_quantize test_pipeline test_acceptance; do
  r=$(PYTHONPATH="$ROOT/tools/ref_shim:$ROOT" timeout 900 python -m pytest -q -p no:cacheprovider "$m.py" 2>&1 | tail -1)
  echo "$m: $r"
done
