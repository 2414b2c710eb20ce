#!/bin/bash
# Round-2 record of one build: GPU tests, ncu --set full of the C5 / C4 / w10
# kernels (limiter counters into profiles/ncu_metrics.json on the box, with the
# library's sha256, BEFORE the bench so its line carries them), bench.py both
# arms (default C5), the other configs (product arm), the launch list, smoke().
#   gpu_record_r02j.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-r02j}
LIB=paper_1810_11518_b200/libaldp_b200.so
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
cp profiles/ncu_metrics.json gpurun_out/ncu_metrics_before.json 2>/dev/null
cap() {  # name, kernel regex, pixels per launch, bench args
  local name=$1 kre=$2 px=$3; shift 3
  local CMD="python bench.py $* --steps 1 --warmup 3 --no-cpu --no-e2e"
  $CMD > gpurun_out/${T}_${name}_plain.json 2> gpurun_out/${T}_${name}_plain.err && \
  ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$kre -s 3 -c 1 \
      -o gpurun_out/${T}_${name} $CMD > gpurun_out/${T}_${name}_ncu.log 2>&1
  echo "$name ncu rc=$?"
  python tools/ncu_to_json.py gpurun_out/${T}_${name}.ncu-rep $name $px $LIB > /dev/null
  python tools/ncu_brief.py gpurun_out/${T}_${name}.ncu-rep > gpurun_out/${T}_ncu_${name}.txt 2>&1
  ncu -i gpurun_out/${T}_${name}.ncu-rep --page source --csv --print-source sass > /tmp/src_${name}.csv 2>/dev/null && \
    python tools/sass_regions.py /tmp/src_${name}.csv 10 >> gpurun_out/${T}_ncu_${name}.txt
}
cap c5 ldp_fast_kernelILi3ELi2ELb1ELb1ELb1ELb0ELi5E 5096079360 --config c5 --images 16384
cap c4 ldp_fast_kernelILi3ELi2ELb1ELb1ELb1ELb0ELi5E 268435456 --config c4
cap w10 ldp_fast_kernelILi3ELi2ELb1ELb1ELb1ELb0ELi16E 642252800 --config w10
rm -f gpurun_out/${T}_c4.ncu-rep  # (64 MiB merge limit: the C4 counters stay in the txt/json)
cp profiles/ncu_metrics.json gpurun_out/ncu_metrics.json
python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?"
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
for c in c2 c3 c4 c5lbp w10 w25; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu >> gpurun_out/${T}_configs.jsonl 2> gpurun_out/${T}_cfg_$c.err; echo "$c rc=$?"
done
python bench.py --force-dist --images 8192 --no-cpu --no-e2e > gpurun_out/${T}_bench_dist1.json 2> gpurun_out/${T}_bench_dist1.err; echo "dist1 rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_launches.log 2>&1; echo "launches rc=$?"
