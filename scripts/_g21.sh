timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g21_pytest.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/g21_pytest.log
timeout 200 python scripts/repro_small.py > gpurun_out/g21_repro.log 2>&1; echo "repro rc $?"; tail -1 gpurun_out/g21_repro.log
timeout 300 python - <<'PY' > gpurun_out/g21_scan.log 2>&1
import sys, time; sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
import synth_instances as SI
for spec in [SI.CONFIG1, SI.SynthSpec(2_000_000, 2000, theta_num=1, theta_den=1), SI.SynthSpec(600_000, 5000)]:
    dev = S.DeviceInstance.from_spec(spec)
    for r in range(3):
        bc, cost, order = S.arrival_queue(dev)
    rep = S.greedy_solve(dev)
    t = rep.timings.row_scan_ns
    print(spec.n, spec.k, "row scan ms", t / 1e6, "GB/s", spec.n * spec.k * 4 / t, flush=True)
    dev.close()
PY
cat gpurun_out/g21_scan.log
