#!/bin/bash
# short timing of the C5-shaped subset and C4, no profiler; optional pytest
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ "$1" == "test" ]; then
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
for args in "--config c5 --images 8192" "--config c4" "--config c3"; do
timeout 300 python bench.py $args --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -5 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$args', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])"
done
