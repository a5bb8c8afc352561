#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/h_pytest.log
timeout 150 python scripts/stress.py 120 > gpurun_out/h_stress.log 2>&1; echo "rc $?" >> gpurun_out/h_stress.log
tail -3 gpurun_out/h_pytest.log; tail -2 gpurun_out/h_stress.log
timeout 1500 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench rc $?" >> gpurun_out/h_bench.err
cat gpurun_out/h_bench.json; tail -3 gpurun_out/h_bench.err
