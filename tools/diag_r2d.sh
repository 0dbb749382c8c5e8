mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "batch or interleaved or m0 or prefix" > gpurun_out/d4_pytest_batch.txt 2>&1
for c in large centrality high-rank mid; do timeout 300 python tools/time_batch.py $c 4 >> gpurun_out/d4_batch.jsonl 2>> gpurun_out/d4_batch.err; done
timeout 300 python tools/time_batch.py large 2 >> gpurun_out/d4_batch.jsonl 2>> gpurun_out/d4_batch.err
timeout 300 python tools/time_batch.py large 8 >> gpurun_out/d4_batch.jsonl 2>> gpurun_out/d4_batch.err
