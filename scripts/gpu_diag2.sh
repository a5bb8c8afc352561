#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/dropin_cases.py 11 gpu > gpurun_out/e_case11.log 2>&1; echo "rc $?" >> gpurun_out/e_case11.log
for seed in 1 2 3; do LBDD_B200_DEBUG=1 timeout 150 python scripts/gpu_big.py 100000 1000 3 $seed >> gpurun_out/e_rep.log 2>&1; echo "rc $?" >> gpurun_out/e_rep.log; done
LBDD_B200_DEBUG=1 LBDD_B200_CHECK=1 timeout 300 python scripts/gpu_big.py 100000 1000 1 20250 >> gpurun_out/e_check.log 2>&1; echo "rc $?" >> gpurun_out/e_check.log
grep -h "rep\|rc\|case" gpurun_out/e_*.log | cut -c1-200
