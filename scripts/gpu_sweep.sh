#!/bin/bash
# knob sweep at 300K x 1000: LBDD_B200_CHUNK values given as args
mkdir -p gpurun_out
for c in "$@"; do LBDD_B200_CHUNK=$c timeout 150 python scripts/gpu_big.py 300000 1000 1 20250 > gpurun_out/sw_chunk$c.log 2>&1; echo "chunk $c: $(grep -o 'objective [0-9]* [0-9.]*s' gpurun_out/sw_chunk$c.log)"; grep -o "'T3': [0-9]*" gpurun_out/sw_chunk$c.log; done
