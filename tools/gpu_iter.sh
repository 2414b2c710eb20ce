#!/bin/bash
# iteration run: GPU parity tests (fast kernel files), then interleaved A/B of
# library variants on C5 (8192 frames), C4 and C3.  gpu_iter.sh LIB...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
[ -z "$SKIP_TESTS" ] && tail -3 gpurun_out/pytest_gpu.log
for args in "--config c5 --images 8192" "--config c4" "--config c3"; do
for rep in 1 2; do
for lib in "$@"; do
if [ "$lib" == "default" ]; then L=""; else L="ALDP_LIB=$lib"; fi
env $L timeout 300 python bench.py $args --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -3 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$lib', '$args', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'], d['config'].get('checksums',{}).get('hist_weighted_sum'))"
done; done; done
