# k_light tile interleave: outermost bands whose tiles interleave by angle (HRG_TILE_MIX)
for m in 0 2 3 4 5 6 8; do echo "mix $m"; HRG_TILE_MIX=$m REPS=5 python tools/ab.py | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['m'], d['t_build_ms'], d['t_light_ms'], d['t_heavy_ms'], d['t_compact_ms'], d['t_rowsort_ms'], d['total_ms'])"; done
