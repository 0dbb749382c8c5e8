mkdir -p gpurun_out
for v in "" "STTSV_HOT=0" "STTSV_HOT=64" "STTSV_CHUNK=1 STTSV_GUIDED=8"; do echo "== mid $v" >> gpurun_out/d1_mid_ab.log; env $v timeout 300 python tools/time_apply.py mid 50 >> gpurun_out/d1_mid_ab.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/d1_launches_mid.csv python tools/profile_edge.py mid 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/d1_launches_mid.csv > gpurun_out/d1_launches_mid.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:edge_kernel -s 2 -c 1 -o gpurun_out/d1_edge_mid python tools/profile_edge.py mid 4 > gpurun_out/d1_ncu_mid.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:edge_kernel -s 2 -c 1 -o gpurun_out/d1_edge_hr python tools/profile_edge.py high-rank 4 > gpurun_out/d1_ncu_hr.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:edge_kernel -s 1 -c 1 -o gpurun_out/d1_edge_batch FUSED=1 python tools/profile_batch.py large > gpurun_out/d1_ncu_batch.log 2>&1
