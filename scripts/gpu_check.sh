#!/bin/bash
# correctness gate + timing after an engine change: tag = $1
tag=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
tail -2 gpurun_out/${tag}_pytest.log
timeout 200 python scripts/repro_small.py > gpurun_out/${tag}_repro.log 2>&1; echo "repro rc $?" >> gpurun_out/${tag}_repro.log
tail -2 gpurun_out/${tag}_repro.log
timeout 200 python scripts/stress.py 150 > gpurun_out/${tag}_stress.log 2>&1; tail -1 gpurun_out/${tag}_stress.log
timeout 120 python scripts/gpu_big.py 100000 1000 1 20250 > gpurun_out/${tag}_100k.log 2>&1; cut -c1-400 gpurun_out/${tag}_100k.log
if [ "$2" = "big" ]; then timeout 400 python scripts/gpu_big.py 1000000 1000 1 20250 > gpurun_out/${tag}_1m.log 2>&1; cut -c1-600 gpurun_out/${tag}_1m.log; fi
