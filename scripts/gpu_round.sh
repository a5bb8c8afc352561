#!/bin/bash
# One GPU-box pass: parity suite, bench, launch list of the bench under ncu.
# usage: scripts/gpu_round.sh [tag]   (outputs under gpurun_out/)
tag=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?" >> gpurun_out/${tag}_bench.err
tail -3 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err
