mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "batch or interleaved or m0 or prefix" > gpurun_out/d3_pytest_batch.txt 2>&1
for c in large centrality high-rank mid; do timeout 300 python tools/time_batch.py $c 4 >> gpurun_out/d3_batch.jsonl 2>> gpurun_out/d3_batch.err; done
timeout 300 python tools/time_batch.py large 2 >> gpurun_out/d3_batch.jsonl 2>> gpurun_out/d3_batch.err
for v in base e4 e2; do bash tools/ab_run.sh d3_mid_ab.log mid:$v; done
