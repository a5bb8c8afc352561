#!/bin/bash
# Correctness gate after an engine change (run under gpurun): the GPU parity
# suite (incl. the reference goldens at scale and the configs[1] checkpoint
# prefix), the random tiny-instance sweep, the mid-size stress loop, and the
# 200K x 1000 phase profile (objective 5246586 on the unchanged engine).
#   scripts/gpu_gate.sh TAG
tag=${1:-gate}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log; tail -3 gpurun_out/${tag}_pytest.log
timeout 200 python scripts/repro_small.py > gpurun_out/${tag}_repro.log 2>&1
echo "repro rc $?" >> gpurun_out/${tag}_repro.log; tail -2 gpurun_out/${tag}_repro.log
timeout 200 python scripts/stress.py 150 > gpurun_out/${tag}_stress.log 2>&1; tail -1 gpurun_out/${tag}_stress.log
timeout 300 python scripts/engine_profile.py --n 200000 > gpurun_out/${tag}_prof.log 2>&1
echo "profile rc $?" >> gpurun_out/${tag}_prof.log; cat gpurun_out/${tag}_prof.log
