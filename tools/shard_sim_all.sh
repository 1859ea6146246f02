# shard simulation of configs 2 and 3 at N = 1, 2, 4, 8 -> gpurun_out/ev/shard_sim.jsonl
out=gpurun_out/ev; mkdir -p $out; rm -f $out/shard_sim.jsonl
for cfg in 2 3; do for n in 1 2 4 8; do
  python bench.py --config $cfg --shard-sim $n --steps 5 >> $out/shard_sim.jsonl 2>> $out/shard_sim.err
done; done
python - <<PY
import json
for l in open("$out/shard_sim.jsonl"):
    d=json.loads(l); print(d["metric"], d["simulated_n_gpus"], round(d["ms_per_step_max"],3), [round(s["ms_per_step"],2) for s in d["shards"]])
PY
