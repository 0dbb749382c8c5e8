#!/bin/bash
# ncu launch lists (per-kernel durations, cold-cache serialised) of a few applies per config:
#   tools/launch_lists.sh TAG cfg1 cfg2 ...   -> gpurun_out/TAG_<cfg>_launches.{csv,txt}
tag=$1; shift
mkdir -p gpurun_out
for cfg in $*; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/${tag}_${cfg}_launches.csv python tools/time_apply.py $cfg 3 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/${tag}_${cfg}_launches.csv > gpurun_out/${tag}_${cfg}_launches.txt 2>&1
done
