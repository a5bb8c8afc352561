#!/bin/bash
# A/B of engine variants (LBDD_B200_LIB) and launch chunk sizes on 200K x 1000
tag=${1:-ab}
mkdir -p gpurun_out
for v in "$@"; do
  [ "$v" = "$tag" ] && continue
  lib=${v%%:*}; specs=${v#*:}
  echo "== $lib" >> gpurun_out/${tag}.log
  LBDD_B200_LIB=$lib timeout 600 python scripts/gpu_delta2.py 200000 1000 ${specs//;/ } >> gpurun_out/${tag}.log 2>&1
done
cut -c1-400 gpurun_out/${tag}.log
