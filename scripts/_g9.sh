timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g9_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g9_pytest.log; tail -3 gpurun_out/g9_pytest.log
timeout 200 python scripts/repro_small.py > gpurun_out/g9_repro.log 2>&1; echo "repro rc $?"; tail -1 gpurun_out/g9_repro.log
LBDD_B200_PROF=1 python scripts/solve_one.py --n 200000 > gpurun_out/g9_200k_prof.log 2>&1; cut -c1-3000 gpurun_out/g9_200k_prof.log
