#!/bin/bash
# engine iteration: parity gate, then 200K x 1000 timing with and without the phase clock
tag=${1:-i}
mkdir -p gpurun_out
timeout 150 python scripts/stress.py 90 > gpurun_out/${tag}_stress.log 2>&1; echo "rc $?" >> gpurun_out/${tag}_stress.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
tail -2 gpurun_out/${tag}_stress.log; tail -3 gpurun_out/${tag}_pytest.log
LBDD_B200_PROF=0 timeout 300 python scripts/gpu_delta2.py 200000 1000 1,1 > gpurun_out/${tag}_t200k.log 2>&1
LBDD_B200_PROF=1 timeout 300 python scripts/gpu_delta2.py 200000 1000 1,1 >> gpurun_out/${tag}_t200k.log 2>&1
cut -c1-200 gpurun_out/${tag}_t200k.log
