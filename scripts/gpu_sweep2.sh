#!/bin/bash
# Δ sweep (cycle/repair, path) on 200K x 1000, then one full ncu capture of a
# late engine launch of the same instance
tag=${1:-s1}
mkdir -p gpurun_out
timeout 900 python scripts/gpu_delta2.py 200000 1000 1,1 1,2 1,4 1,16 1,0 2,2 4,4 > gpurun_out/${tag}_delta.log 2>&1
cat gpurun_out/${tag}_delta.log | cut -c1-600
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster_engine -s 30 -c 1 \
  -o gpurun_out/${tag}_engine python scripts/ncu_step.py 200000 1000 > gpurun_out/${tag}_ncu_engine.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/${tag}_ncu_engine.log
