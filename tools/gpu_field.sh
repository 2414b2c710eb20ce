#!/bin/bash
# One gpurun call: full GPU test suite, the rank-2 field/verify bench, and an
# ncu capture of the int16 response-field kernel.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/field_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/field_tests.log
python tools/bench_field.py > gpurun_out/field_bench.jsonl 2> gpurun_out/field_bench.err && \
ncu --set full --clock-control none --import-source on -k regex:response_field_kernel -c 1 \
    -o gpurun_out/ncu_field16 -f python tools/bench_field.py --images 256 --steps 1 --warmup 0 \
    > gpurun_out/ncu_field.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"response_field|verify" -c 20 --csv \
    --log-file gpurun_out/field_launches.csv python tools/bench_field.py --images 256 --steps 2 --warmup 1 \
    > gpurun_out/ncu_field_launch.log 2>&1
tail -3 gpurun_out/field_tests.log; cat gpurun_out/field_bench.jsonl
