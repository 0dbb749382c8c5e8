set -e
python tools/variants.py 8 base: i16:-DSTTSV_ID16=1 i16e6:-DSTTSV_ID16=1,-DSTTSV_EPL=6 i16n8:-DSTTSV_ID16=1,-DSTTSV_NCW_ID16=8 i16n10:-DSTTSV_ID16=1,-DSTTSV_NCW_ID16=10 > gpurun_out/r1_var59_build.log 2>&1
for r in 1 2; do for v in base i16 i16e6 i16n8 i16n10; do STTSV_LIB_PATH=build/variants/libsttsv_$v.so python tools/time_apply.py large 30 | sed "s/^/$v /"; done; done
STTSV_LIB_PATH=build/variants/libsttsv_i16.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_bucket or configs_reduced or fuzz or random_buckets or scatter" 2>&1 | tail -5
