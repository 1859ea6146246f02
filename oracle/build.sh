#!/bin/sh
# Builds the CPU oracle (test infrastructure only; see hrg_oracle.h).
set -e
cd "$(dirname "$0")"
gcc -O2 -std=gnu11 -fPIC -shared -fopenmp -ffp-contract=off -fno-fast-math \
    -o libhrg_oracle.so hrg_oracle.c -lquadmath -lm
