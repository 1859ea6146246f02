#!/bin/bash
# Evidence for profiles/ (run on the GPU box): bench lines, sweep, shard-sim,
# launch list, ncu captures of the dominant kernels.  Output: gpurun_out/ev/
set -x
out=gpurun_out/ev; mkdir -p $out
python bench.py > $out/bench_config2.json 2> $out/bench_config2.err
python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err
python bench.py --config 1 > $out/bench_config1.json 2> $out/bench_config1.err
python bench.py --config 3 --no-cpu-baseline --no-parity --steps 5 > $out/bench_config3.json 2> $out/bench_config3.err
python bench.py --sweep > $out/sweep_config4.jsonl 2> $out/sweep.err
for cfg in 2 3; do for n in 1 2 4 8; do
  python bench.py --config $cfg --shard-sim $n --steps 5 >> $out/shard_sim.jsonl 2>> $out/shard_sim.err
done; done
python tools/prof_gen.py > $out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_config2_sample.csv python tools/prof_gen.py > $out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_light|k_compact_light' --launch-skip 2 --launch-count 2 -o $out/ncu_full_config2 -f python tools/prof_gen.py > $out/ncu_full.log 2>&1
ls -la $out
