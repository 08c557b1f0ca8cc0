#!/bin/bash
# cold-step graph timing per variant: tools/exp_cold.sh "CFGS" VARIANT...
cfgs=$1; shift
for v in "$@"; do
  if [ "$v" = main ]; then lib=paper_1305_3122_b200/libfemasm_b200.so; else lib=tools/exp/lib_$v.so; fi
  for c in $cfgs; do
    echo "== $v $c"; FEMASM_B200_LIB=$lib timeout 300 python tools/cold_time.py $c 2>&1 | grep -v Warning
  done
done
