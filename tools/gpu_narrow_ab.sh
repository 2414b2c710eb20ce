#!/bin/bash
# narrow-cell A/B: GPU narrow tests, then w10 / w25 with owned tiling off / on
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "narrow" > gpurun_out/pytest_narrow.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_narrow.log
for c in w10 w25; do for rep in 1 2; do for own in 0 1 2; do
ALDP_NARROW_HIST=$own timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -3 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$c own=$own', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['ms_per_step'], d['config'].get('checksums',{}).get('hist_weighted_sum'))"
done; done; done
