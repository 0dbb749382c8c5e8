#!/bin/bash
# A/B of the TMA ring size (STTSV_RING_KB) and the 16-bit-id tile size (STTSV_EPL16) on mid
# (N = 10) and large (N = 8): a smaller ring leaves more of the SM's 256 KB to L1, which
# caches the series-table rows the DP gathers.  Variants built by tools/variants.py.
mkdir -p gpurun_out
out=gpurun_out/r2_ab_ring.log
: > $out
for rep in 1 2; do
  for spec in mid:base mid:m_r108e4 mid:m_r80e4 mid:m_r64e4 mid:m_r48e2 large:base large:l_r108e4 large:l_r80e6 large:l_r80e4 large:l_r64e4; do
    cfg=${spec%%:*}; lib=${spec#*:}
    if [ "$lib" = base ]; then
      timeout 300 python tools/time_apply.py $cfg 20 2>&1 | grep step_ms | sed "s/^/$lib /" >> $out
    elif [ -f build/variants/libsttsv_$lib.so ]; then
      STTSV_LIB_PATH=build/variants/libsttsv_$lib.so timeout 300 python tools/time_apply.py $cfg 20 2>&1 | grep step_ms | sed "s/^/$lib /" >> $out
    fi
  done
done
cat $out
