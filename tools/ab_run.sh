#!/bin/bash
# A/B timing of library variants on the GPU box: tools/ab_run.sh OUT "cfg:lib cfg:lib ..."
# (lib = a name under build/variants/ or "base" for the in-tree libsttsv.so; WAITPROF
# variants print the per-class consumer cycles)
out=$1; shift
mkdir -p gpurun_out
for spec in $*; do
  cfg=${spec%%:*}; lib=${spec#*:}
  if [ "$lib" = base ]; then
    WAITPROF_CLASSES=1 timeout 300 python tools/time_apply.py $cfg 20 >> gpurun_out/$out 2>&1
  else
    STTSV_LIB_PATH=build/variants/libsttsv_$lib.so WAITPROF_CLASSES=1 timeout 300 python tools/time_apply.py $cfg 20 >> gpurun_out/$out 2>&1
  fi
done
