# sharded light pass: the per-query candidate limit of the light pass (HRG_LIGHT_MAX)
for lm in 2048 1024 512 256 128; do echo "shard 1/8 light_max=$lm"; HRG_LIGHT_MAX=$lm SK=1 SN=8 REPS=6 python tools/shard_gen.py; done
for lm in 2048 1024 512 256; do echo "shard 1/2 light_max=$lm"; HRG_LIGHT_MAX=$lm SK=1 SN=2 REPS=6 python tools/shard_gen.py; done
for lm in 2048 1024 512; do echo "unsharded light_max=$lm"; HRG_LIGHT_MAX=$lm REPS=5 python tools/ab.py | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['m'], d['heavy'], d['t_light_ms'], d['t_heavy_ms'], d['t_compact_ms'], d['t_rowsort_ms'], d['total_ms'])"; done
