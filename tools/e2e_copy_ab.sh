# result-copy variants, libraries alternating: usage e2e_copy_ab.sh "f f f" lib lib ...
fr=$1; shift
for rep in 1 2 3; do for lib in "$@"; do
  if [ "$lib" = "default" ]; then l=""; else l="exp/lib_$lib.so"; fi
  HRGEN_B200_LIB=$l python tools/e2e_copy_ab.py $fr; done; done
