LBDD_B200_PROF=1 python scripts/solve_one.py --n 200000 > gpurun_out/g5_200k_prof.log 2>&1; cut -c1-3000 gpurun_out/g5_200k_prof.log
