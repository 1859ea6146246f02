#!/bin/bash
# usage: tools/ab_run.sh out.jsonl variant...   (env N K G SEED ORDER pass through)
out=$1; shift
for v in "$@"; do
  if [ "$v" = "default" ]; then lib=""; else lib="exp/lib_$v.so"; fi
  HRGEN_B200_LIB=$lib timeout 300 python tools/ab.py >> $out 2>&1 || echo "{\"lib\": \"$v\", \"failed\": true}" >> $out
done
