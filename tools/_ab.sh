for c in large centrality mid tiny; do python tools/time_apply.py $c 30; done > gpurun_out/r1_v56_time.log 2>&1
python tools/variants.py 8 e6: e8:-DSTTSV_EPL16=8 e7:-DSTTSV_EPL16=7 > gpurun_out/r1_var61_build.log 2>&1
for r in 1 2; do for v in e6 e8 e7; do STTSV_LIB_PATH=build/variants/libsttsv_$v.so python tools/time_apply.py large 30 | sed "s/^/$v /"; done; done > gpurun_out/r1_var61.log 2>&1
VARIANTS_KEEP=1 python tools/variants.py 12 c6: c5:-DSTTSV_EPL16=5 c4:-DSTTSV_EPL16=4 c8:-DSTTSV_EPL16=8 > gpurun_out/r1_var62_build.log 2>&1
for r in 1 2; do for v in c6 c5 c4 c8; do STTSV_LIB_PATH=build/variants/libsttsv_$v.so python tools/time_apply.py centrality 30 | sed "s/^/$v /"; done; done > gpurun_out/r1_var62.log 2>&1
