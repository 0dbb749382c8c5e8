mkdir -p gpurun_out
export FUSED=1
timeout 300 python tools/profile_batch.py large 4 > gpurun_out/d2_batch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:edge_kernel -s 1 -c 1 -o gpurun_out/d2_edge_batch python tools/profile_batch.py large 4 > gpurun_out/d2_ncu_batch.log 2>&1
unset FUSED
timeout 600 ncu --set full --clock-control none --import-source on -k regex:edge_kernel -s 2 -c 1 -o gpurun_out/d2_edge_large python tools/profile_edge.py large 4 > gpurun_out/d2_ncu_large.log 2>&1
