#!/bin/bash
# Round-2 record: GPU tests, bench.py both arms (default C5), the NCCL path at
# world size 1 (uint16 wire), launch list of the default bench, and one ncu
# --set full capture of the C5 cell kernel (16384 frames = one launch).
#   gpu_record_r02.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-r02}
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?"
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python bench.py --force-dist --images 8192 --no-cpu --no-e2e > gpurun_out/${T}_bench_dist1.json 2> gpurun_out/${T}_bench_dist1.err; echo "dist1 rc=$?"
CMD="python bench.py --config c5 --images 16384 --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/${T}_ncu_plain.json 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ldp_fast_kernelILi3ELi2ELb1ELb1ELb1 -s 3 -c 1 -o gpurun_out/${T}_c5 $CMD > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_launches.log 2>&1; echo "launches rc=$?"
