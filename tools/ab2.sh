#!/bin/bash
# A/B on two configs: bash tools/ab2.sh "A.so B.so" "--config c2"
cd "$(dirname "$0")/.."
bash tools/ab.sh $1 -- --steps 3 --warmup 3
bash tools/ab.sh $1 -- --steps 3 --warmup 3 $2
