#!/bin/bash
# Correctness gate after an engine change (run under gpurun): the GPU parity
# suite, the random tiny-instance sweep, the mid-size stress loop, and one
# timed solve (default 100K x 1000 against its reference golden).
#   scripts/gpu_gate.sh TAG [GOLDEN]
tag=${1:-gate}
golden=${2:-k1000_n100k}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log; tail -3 gpurun_out/${tag}_pytest.log
timeout 200 python scripts/repro_small.py > gpurun_out/${tag}_repro.log 2>&1
echo "repro rc $?" >> gpurun_out/${tag}_repro.log; tail -2 gpurun_out/${tag}_repro.log
timeout 200 python scripts/stress.py 150 > gpurun_out/${tag}_stress.log 2>&1; tail -1 gpurun_out/${tag}_stress.log
timeout 600 python scripts/solve_one.py --golden $golden > gpurun_out/${tag}_solve.log 2>&1
echo "solve rc $?" >> gpurun_out/${tag}_solve.log; cut -c1-600 gpurun_out/${tag}_solve.log
