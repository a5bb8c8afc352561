"""TEST INFRASTRUCTURE ONLY -- the reference's CPU time profile of the
configs[1] solve, for bench.py's calibrated CPU baseline.

Inputs (build container): the progress log of oracle/run_ref_scale.py's
full configs[1] run (cumulative seconds every `mark` arrivals) and one of its
checkpoints (the centers of the first X arrivals, in arrival order). Output:
profiles/ref_cpu_profile_configs1.json and the checkpoint, zlib-compressed,
under tests/golden/ckpt/. Also times, here and now, the two samples bench.py
times on the GPU box (first --first arrivals from scratch; --arrivals
arrivals resumed from the checkpoint), so the box/here speed ratio can be
applied to the profile.

    python oracle/make_cpu_profile.py --log /root/refruns/config1_full.log \
        --ckpt /root/refruns/config1_ckpt_25000.i16
"""
import argparse
import json
import os
import re
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--log", required=True)
    p.add_argument("--ckpt", required=True)
    p.add_argument("--first", type=int, default=300)
    p.add_argument("--arrivals", type=int, default=40)
    a = p.parse_args()
    import bench
    import synth_instances as SI
    spec = SI.CONFIG1
    marks = []
    every = None
    for line in open(a.log):
        m = re.match(r"\[ref\] (\d+) arrivals ([\d.]+) s", line)
        if m:
            cnt, t = int(m.group(1)), float(m.group(2))
            if every is None:
                every = cnt
            marks.append(t)
    cs = np.fromfile(a.ckpt, dtype=np.int16)
    x_ck = len(cs)
    prob = SI.problem(spec)
    rs = bench.RefSampler(prob)
    t_first, setup_s, nfirst = rs.first(a.first)
    ck_setup = rs.open_checkpoint(cs)
    t_st, nst = rs.steady(a.arrivals)
    rs.close()
    # the log's times include the run's setup (arrival queue + empty index);
    # profile marks are loop seconds
    loop_marks = [round(m - setup_s, 2) for m in marks]
    t_ck_here = loop_marks[x_ck // every - 1]
    name = f"config1_{x_ck}.i16.z"
    with open(os.path.join(ROOT, "tests", "golden", "ckpt", name), "wb") as f:
        f.write(zlib.compress(cs.tobytes(), 9))
    out = {
        "spec": spec.name(), "n": spec.n, "mark_every": every, "marks_s": loop_marks,
        "setup_s_here": round(setup_s, 2),
        "checkpoint": {"file": name, "arrivals": x_ck, "loop_s_here": t_ck_here,
                       "resume_setup_s_here": round(ck_setup, 2)},
        "here": {"first_arrivals": nfirst, "first_loop_s": round(t_first, 3),
                 "steady_arrivals": nst, "steady_s_per_arrival": round(t_st / max(nst, 1), 4),
                 "host": os.uname().nodename, "cpu": open("/proc/cpuinfo").read().split(
                     "model name")[1].split(":")[1].split("\n")[0].strip(),
                 "note": "measured in the build container while the full run and other "
                         "reference runs shared its 8 cores (the same conditions as the marks)"},
        "source": "oracle/run_ref_scale.py --tag config1_full (oracle/_ref/liblbdd_ref.so, "
                  "-O3 -DNDEBUG, sequential asral loop of solver.hpp:143-166)",
        "made": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    with open(os.path.join(ROOT, "profiles", "ref_cpu_profile_configs1.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out)[:600])


if __name__ == "__main__":
    main()
