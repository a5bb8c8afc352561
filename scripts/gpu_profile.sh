#!/bin/bash
# Measurement pass (run under gpurun, one GPU): the bench line, then -- each
# only after its plain command exited 0 -- the ncu launch list of one solve
# and --set full captures of the scans and of one engine launch.
#   scripts/gpu_profile.sh TAG [N] [ENGINE_LAUNCH_TO_SKIP]
tag=${1:-prof}
N=${2:-1000000}
mkdir -p gpurun_out
timeout 1700 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc $?" >> gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_bench.json
timeout 400 python scripts/solve_one.py --n $N --scan > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/${tag}_plain.log; exit 1; }
cut -c1-400 gpurun_out/${tag}_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
  --log-file gpurun_out/${tag}_launches.csv python scripts/solve_one.py --n $N --scan > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launch list rc $?"; python scripts/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launch_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_argmin|row_argmin" -c 3 \
  -o gpurun_out/${tag}_scans python scripts/solve_one.py --n $N --scan > gpurun_out/${tag}_ncu_scans.log 2>&1
echo "scans rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cluster_engine -s ${3:-150} -c 1 \
  -o gpurun_out/${tag}_engine python scripts/solve_one.py --n $N > gpurun_out/${tag}_ncu_engine.log 2>&1
echo "engine rc $?"
