#!/bin/bash
# experiment round on the GPU box: tools/exp_run.sh "CFGS" VARIANT... (variant "main" = in-tree library)
# per variant: quick_time over CFGS, then the C1/C2/EL64 reference-digest tests
cfgs=$1; shift
for v in "$@"; do
  if [ "$v" = main ]; then lib=paper_1305_3122_b200/libfemasm_b200.so; else lib=tools/exp/lib_$v.so; fi
  echo "== $v"
  FEMASM_B200_LIB=$lib timeout 300 python tools/quick_time.py $cfgs 2>&1 | grep -v Warning
  FEMASM_B200_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "test_reference_digests and not large" 2>&1 | tail -1
done
