#!/bin/bash
# bench line, then ncu engine profile (one launch) of the bench step
tag=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?" >> gpurun_out/${tag}_bench.err
cat gpurun_out/${tag}_bench.json
timeout 280 python scripts/ncu_step.py 1000000 1000 > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cluster_engine -s 150 -c 1 \
  -o gpurun_out/${tag}_engine python scripts/ncu_step.py 1000000 1000 > gpurun_out/${tag}_ncu_engine.log 2>&1
echo "engine rc $?"; cat gpurun_out/${tag}_plain.log
