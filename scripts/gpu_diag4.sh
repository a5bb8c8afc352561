#!/bin/bash
# after the reconstruct race fix: parity suite, stress, 1M determinism, tuning knobs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g_pytest.log
timeout 150 python scripts/stress.py 120 > gpurun_out/g_stress.log 2>&1; echo "rc $?" >> gpurun_out/g_stress.log
for D in 1 4 16; do LBDD_B200_DELTA=$D timeout 100 python scripts/gpu_big.py 100000 1000 1 20250 > gpurun_out/g_delta$D.log 2>&1; done
LBDD_B200_LIB=$PWD/paper_2304_06543_b200/lib_t512/liblbdd_b200.so timeout 100 python scripts/gpu_big.py 100000 1000 1 20250 > gpurun_out/g_t512.log 2>&1
timeout 500 python scripts/gpu_big.py 1000000 1000 2 20250 > gpurun_out/g_big.log 2>&1; echo "rc $?" >> gpurun_out/g_big.log
tail -3 gpurun_out/g_pytest.log; tail -2 gpurun_out/g_stress.log; grep -h "rep\|lib" gpurun_out/g_delta*.log gpurun_out/g_t512.log gpurun_out/g_big.log | cut -c1-150
