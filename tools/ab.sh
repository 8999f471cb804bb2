#!/bin/bash
# A/B timing of two library builds in one GPU session (box-to-box variation
# is ~5%): tools/ab.sh WORKLOAD REPS LIB_A LIB_B  -> gpurun_out/ab.log
w=$1; n=$2; shift 2
rm -f gpurun_out/ab.log
for i in $(seq $n); do for L in "$@"; do
  echo "lib $L" >> gpurun_out/ab.log
  DFM_LIB=$PWD/$L python tools/split_bench.py --workload $w --steps 15 >> gpurun_out/ab.log 2>&1
done; done
