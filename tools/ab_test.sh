#!/bin/bash
# GPU parity tests against an A/B variant build, then the A/B bench.
# usage (through gpurun): bash tools/ab_test.sh VARIANT.so [OTHER.so ...] [-- bench args]
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
MPM_B200_LIB="$PWD/variants/$1" timeout 420 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
bash tools/ab.sh "$@"
