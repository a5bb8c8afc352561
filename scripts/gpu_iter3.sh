#!/bin/bash
# paired relax: parity gate, then A/B timing on 200K x 1000 (LBDD_B200_PAIRS=0 / 1)
tag=${1:-i}
mkdir -p gpurun_out
timeout 150 python scripts/stress.py 100 > gpurun_out/${tag}_stress.log 2>&1; echo "rc $?" >> gpurun_out/${tag}_stress.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
tail -2 gpurun_out/${tag}_stress.log; tail -3 gpurun_out/${tag}_pytest.log
LBDD_B200_PAIRS=0 timeout 300 python scripts/gpu_delta2.py 200000 1000 1,1 > gpurun_out/${tag}_t200k.log 2>&1
LBDD_B200_PAIRS=1 timeout 300 python scripts/gpu_delta2.py 200000 1000 1,1 >> gpurun_out/${tag}_t200k.log 2>&1
cut -c1-120 gpurun_out/${tag}_t200k.log
