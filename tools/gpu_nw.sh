#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest(nw1) rc=$?"; tail -2 gpurun_out/pytest_gpu.log
ALDP_LANE_WORDS=2 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest(nw2) rc=$?"; tail -2 gpurun_out/pytest_gpu2.log
for nw in 1 2; do
for args in "--config c5 --images 8192" "--config c4" "--config c3"; do
ALDP_LANE_WORDS=$nw timeout 300 python bench.py $args --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -5 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('nw=$nw $args', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])"
done; done
