#!/bin/bash
# reference arm (bounded CPU sample) + other-shape solve samples
mkdir -p gpurun_out
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; echo "ref rc $?" >> gpurun_out/f_ref.err
cat gpurun_out/f_ref.json; tail -2 gpurun_out/f_ref.err
timeout 1500 python scripts/gpu_shapes_solve.py > gpurun_out/f_shapes.log 2>&1; echo "shapes rc $?" >> gpurun_out/f_shapes.log
cat gpurun_out/f_shapes.log
