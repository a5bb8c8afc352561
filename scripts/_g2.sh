mkdir -p gpurun_out
python scripts/latency_floor.py
python scripts/solve_one.py --n 200000 > gpurun_out/g2_200k.log 2>&1; cut -c1-1500 gpurun_out/g2_200k.log
LBDD_B200_PROF=1 python scripts/solve_one.py --n 200000 > gpurun_out/g2_200k_prof.log 2>&1; cut -c1-1500 gpurun_out/g2_200k_prof.log
