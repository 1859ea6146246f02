for rep in 1 2 3; do for lib in exp/lib_plain.so ""; do HRGEN_B200_LIB=$lib python tools/e2e_copy_ab.py 1 0.6 0.45 0.3 0.15 0; done; done
