#!/bin/bash
mkdir -p gpurun_out
DROP_IN_VERBOSE=1 timeout 100 oracle/_ref/drop_in_check 12 > gpurun_out/f_dropin.log 2>&1; echo "dropin rc $?" >> gpurun_out/f_dropin.log
LBDD_B200_DEBUG=1 LBDD_B200_CHECK=1 timeout 300 python scripts/gpu_big.py 100000 1000 1 20250 > gpurun_out/f_check.log 2>&1; echo "rc $?" >> gpurun_out/f_check.log
tail -5 gpurun_out/f_dropin.log; cat gpurun_out/f_check.log | cut -c1-300
