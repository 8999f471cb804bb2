#!/bin/bash
# Everything a profiles/rNN directory holds, in one GPU session:
#   tools/profile_round.sh r02d      -> gpurun_out/r02d/
# bench lines for configs 0-4 and the reference arm, the shard scaling, the
# bin kernel's phase trace, the ncu launch list of the bench command and one
# `ncu --set full` capture of the step kernels (numbers printed under ncu are
# never bench values; each ncu pass runs only after its command exited 0).
set -u
r=${1:-rXX}
o=gpurun_out/$r
mkdir -p $o
for w in config1 config0 config2 config3 config4; do
  python bench.py --workload $w > $o/bench_$w.json 2> $o/bench_$w.err || echo "bench $w failed" >> $o/errors.log
done
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_reference.json 2>> $o/errors.log
python tools/shard_bench.py config1 1 2 4 8 > $o/shard_config1.log 2>&1
python tools/shard_bench.py config3 1 2 4 8 > $o/shard_config3.log 2>&1
python tools/trace_bin.py --workload config1 > $o/trace_bin_config1.json 2>&1
python tools/trace_bin.py --workload config1 --shards 8 > $o/trace_bin_config1_shard8.json 2>&1
python tools/wiener_bench.py > $o/wiener.log 2>&1
if python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-init > $o/bench_short.json 2>> $o/errors.log; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/launches_config1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-init > $o/ncu_launches.log 2>&1
fi
if python tools/split_bench.py --workload config1 --steps 3 > $o/split_c1.json 2>> $o/errors.log; then
  ncu --set full --clock-control none --import-source on -k regex:'k_em_bin|k_tupd_mma|k_pdw|k_vupd_mma' \
    --launch-skip 40 --launch-count 4 -o $o/${r}_step_c1 -f \
    python tools/split_bench.py --workload config1 --steps 12 > $o/ncu_step.log 2>&1
fi
ls -la $o
