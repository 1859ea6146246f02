# result-copy variants, alternating: usage e2e_copy_ab.sh "f f f" ENV=VAL ENV=VAL ...   (each its own process)
fr=$1; shift
for rep in 1 2 3; do for v in "$@"; do echo -n "$v  "; env $v python tools/e2e_copy_ab.py $fr; done; done
