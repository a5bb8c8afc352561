#!/bin/bash
# Diagnostics for the 1M x 1000 objective divergence and the drop-in hang.
mkdir -p gpurun_out
DROP_IN_VERBOSE=1 timeout 120 oracle/_ref/drop_in_check 12 > gpurun_out/d_dropin.log 2>&1; echo "dropin rc $?" >> gpurun_out/d_dropin.log
LBDD_B200_DEBUG=1 timeout 300 python scripts/gpu_big.py 1000000 1000 1 > gpurun_out/d_big_new.log 2>&1; echo "rc $?" >> gpurun_out/d_big_new.log
LBDD_B200_LIB=$PWD/paper_2304_06543_b200/lib_old/liblbdd_b200.so timeout 300 python scripts/gpu_big.py 1000000 1000 1 > gpurun_out/d_big_old.log 2>&1; echo "rc $?" >> gpurun_out/d_big_old.log
for n in 100000 300000; do LBDD_B200_DEBUG=1 timeout 200 python scripts/gpu_big.py $n 1000 1 >> gpurun_out/d_mid.log 2>&1; echo "rc $?" >> gpurun_out/d_mid.log; done
timeout 200 python scripts/stress.py 150 > gpurun_out/d_stress.log 2>&1; echo "rc $?" >> gpurun_out/d_stress.log
tail -5 gpurun_out/d_*.log
