#!/bin/bash
# Profiles of one bench step (scripts/ncu_step.py = one configs[1] solve + the
# build_index scan): plain run first, then the launch list, then --set full
# captures of the scans and of one cluster-engine launch.
tag=${1:-r1}
N=${2:-1000000}
mkdir -p gpurun_out
timeout 280 python scripts/ncu_step.py $N 1000 > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/${tag}_plain.log; exit 1; }
cat gpurun_out/${tag}_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
  --log-file gpurun_out/${tag}_launches.csv python scripts/ncu_step.py $N 1000 > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launch list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_argmin|row_argmin" -c 3 \
  -o gpurun_out/${tag}_scans python scripts/ncu_step.py $N 1000 > gpurun_out/${tag}_ncu_scans.log 2>&1
echo "scans rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cluster_engine -s ${3:-150} -c 1 \
  -o gpurun_out/${tag}_engine python scripts/ncu_step.py $N 1000 > gpurun_out/${tag}_ncu_engine.log 2>&1
echo "engine rc $?"
ls -la gpurun_out/
