#!/bin/bash
# round gate + measurement: parity, bench line, launch list, engine ncu capture
tag=${1:-r03}
mkdir -p gpurun_out
timeout 150 python scripts/stress.py 90 > gpurun_out/${tag}_stress.log 2>&1; echo "rc $?" >> gpurun_out/${tag}_stress.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
tail -2 gpurun_out/${tag}_stress.log; tail -3 gpurun_out/${tag}_pytest.log
timeout 1500 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?" >> gpurun_out/${tag}_bench.err
cat gpurun_out/${tag}_bench.json; tail -3 gpurun_out/${tag}_bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python scripts/ncu_step.py 1000000 1000 > gpurun_out/${tag}_ncu_launches.log 2>&1; echo "launches rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster_engine -s 30 -c 1 \
  -o gpurun_out/${tag}_engine python scripts/ncu_step.py 200000 1000 > gpurun_out/${tag}_ncu_engine.log 2>&1
echo "engine ncu rc $?"
