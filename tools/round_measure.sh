#!/bin/bash
# One GPU call's worth of round measurements (tag = version label):
#   tools/round_measure.sh TAG
# GPU tests, the bench line, all five configs, the bench launch list and one
# ncu --set full capture of the large edge kernel (each only after its own
# command ran clean without ncu).  Everything lands in gpurun_out/.
tag=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 python tools/bench_configs.py --out gpurun_out/${tag}_configs.jsonl > gpurun_out/${tag}_configs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_large.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-merge-report --no-batch-report --no-memo-report > gpurun_out/${tag}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launches_large.csv > gpurun_out/${tag}_launches_large.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_kernel -s 2 -c 1 \
  -o gpurun_out/${tag}_edge_large python tools/profile_edge.py large 4 > gpurun_out/${tag}_ncu_full.log 2>&1
