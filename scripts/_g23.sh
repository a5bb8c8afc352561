timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g23_pytest.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/g23_pytest.log
timeout 900 python scripts/solve_one.py --n 400000 --k 2000 --theta 1/1 > gpurun_out/g23_k2000.log 2>&1; echo "k2000 rc $?"; cut -c1-400 gpurun_out/g23_k2000.log
