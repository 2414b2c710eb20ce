#!/bin/bash
# End-of-round record: GPU tests, smoke, the default bench (both arms), the
# LBP and field benches, the ncu launch list of the default bench command and
# full captures of the three dominant kernels. Outputs land in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01e}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/${TAG}_gpu.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/${TAG}_bench.json
timeout 900 python bench.py --config c5lbp --no-cpu > gpurun_out/${TAG}_bench_lbp.json 2> gpurun_out/${TAG}_bench_lbp.err; echo "lbp rc=$?"
timeout 900 python bench.py --config c5lbp --impl reference > gpurun_out/${TAG}_bench_lbp_ref.json 2>&1; echo "lbp ref rc=$?"
timeout 600 python tools/bench_field.py > gpurun_out/${TAG}_field.jsonl 2> gpurun_out/${TAG}_field.err; echo "field rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
B="python bench.py --config c5 --images 4096 --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > gpurun_out/${TAG}_sub.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ldp_fast -s 3 -c 1 -o gpurun_out/${TAG}_full $B > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu-full rc=$?"
L="python bench.py --config c5lbp --images 4096 --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $L > gpurun_out/${TAG}_sub_lbp.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ldp_fast -s 3 -c 1 -o gpurun_out/${TAG}_full_lbp $L > gpurun_out/${TAG}_ncu_full_lbp.log 2>&1; echo "ncu-full-lbp rc=$?"
F="python tools/bench_field.py --images 512 --steps 2 --warmup 1"
timeout 600 $F > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:response_field_row -s 2 -c 1 -o gpurun_out/${TAG}_full_field $F > gpurun_out/${TAG}_ncu_field.log 2>&1; echo "ncu-field rc=$?"
# summarise on the box and drop the .ncu-rep files (gpurun copies back <= 64 MiB)
for r in full full_lbp full_field; do
  [ -f gpurun_out/${TAG}_$r.ncu-rep ] || continue
  L=""; [ "$r" == "full" ] && L=gpurun_out/${TAG}_launches.csv
  python tools/ncu_summary.py gpurun_out/${TAG}_$r.ncu-rep gpurun_out/${TAG}_ncu_$r.md $L > /dev/null 2>&1
  [ "$r" == "full" ] && ncu -i gpurun_out/${TAG}_$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_source_sass.csv 2>/dev/null
  rm -f gpurun_out/${TAG}_$r.ncu-rep
done
du -sh gpurun_out
