#!/bin/bash
# parity gate: GPU tests, driver smoke, random tiny-instance stress
tag=${1:-v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${tag}_smoke.log
timeout 150 python scripts/stress.py 120 > gpurun_out/${tag}_stress.log 2>&1; echo "rc $?" >> gpurun_out/${tag}_stress.log
tail -3 gpurun_out/${tag}_pytest.log; tail -2 gpurun_out/${tag}_smoke.log; tail -2 gpurun_out/${tag}_stress.log
