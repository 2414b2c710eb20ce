#!/bin/bash
# Record run for the SURVEY 8f "next" rows: LBP bench (both arms), the
# response-field / verify bench with an ncu capture of the row kernel, and the
# PGM extract / bench-CSV measurements. Outputs land in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01c}
timeout 900 python bench.py --config c5lbp --impl reference > gpurun_out/${TAG}_lbp_ref.json 2> gpurun_out/${TAG}_lbp_ref.err; echo "lbp ref rc=$?"
timeout 900 python bench.py --config c5lbp > gpurun_out/${TAG}_lbp.json 2> gpurun_out/${TAG}_lbp.err; echo "lbp rc=$?"
timeout 600 python tools/bench_field.py > gpurun_out/${TAG}_field.jsonl 2> gpurun_out/${TAG}_field.err; echo "field rc=$?"
F="python tools/bench_field.py --images 512 --steps 2 --warmup 1"
timeout 600 $F > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:response_field_row -s 2 -c 1 -o gpurun_out/${TAG}_field_full $F > gpurun_out/${TAG}_ncu_field.log 2>&1; echo "ncu field rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_field_launches.csv $F > /dev/null 2>&1; echo "ncu field launches rc=$?"
timeout 900 python tools/bench_io.py --out-dir gpurun_out > gpurun_out/${TAG}_io.jsonl 2> gpurun_out/${TAG}_io.err; echo "io rc=$?"
cat gpurun_out/${TAG}_lbp.json gpurun_out/${TAG}_lbp_ref.json gpurun_out/${TAG}_field.jsonl gpurun_out/${TAG}_io.jsonl | cut -c1-400
