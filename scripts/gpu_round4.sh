#!/bin/bash
# parity gate + bench line
tag=${1:-r04}
mkdir -p gpurun_out
timeout 150 python scripts/stress.py 90 > gpurun_out/${tag}_stress.log 2>&1; echo "rc $?" >> gpurun_out/${tag}_stress.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${tag}_smoke.log
tail -2 gpurun_out/${tag}_stress.log; tail -3 gpurun_out/${tag}_pytest.log; tail -2 gpurun_out/${tag}_smoke.log
grep -q "pytest rc 0" gpurun_out/${tag}_pytest.log || exit 1
timeout 1500 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?" >> gpurun_out/${tag}_bench.err
cat gpurun_out/${tag}_bench.json; tail -3 gpurun_out/${tag}_bench.err
