#!/bin/bash
# GPU test suite only (through gpurun): parity record + pytest -m gpu summary
cd "$(dirname "$0")/.."
O=gpurun_out/tests; mkdir -p $O
python -m paper_1910_00935_b200.build > /dev/null
export MPM_PARITY_RECORD=$O/parity_record.jsonl; rm -f $MPM_PARITY_RECORD
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
tail -4 $O/pytest_gpu.txt
