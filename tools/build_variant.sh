#!/bin/bash
# Experiment builds: tools/build_variant.sh NAME "-DFLAG=1 ..." -> variants/NAME/libqmoe.so
# (load with QMOE_LIB_PATH=variants/NAME/libqmoe.so; the product build is `make` in csrc/)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -C "$ROOT/paper_2310_16795_b200/csrc" -j4 OUT="$ROOT/variants/$1" EXTRA="$2" > /dev/null
echo "$ROOT/variants/$1/libqmoe.so"
