#!/bin/bash
# bench lines only (configs 1-3 + reference arm) -> gpurun_out/ev/
out=gpurun_out/ev; mkdir -p $out
python bench.py > $out/bench_config2.json 2> $out/bench_config2.err
python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err
python bench.py --config 1 > $out/bench_config1.json 2> $out/bench_config1.err
python bench.py --config 3 --no-cpu-baseline --no-parity --steps 5 > $out/bench_config3.json 2> $out/bench_config3.err
python -m pytest tests/test_abi.py tests/test_integration_stub.py -m gpu -q 2>&1 | tail -2
