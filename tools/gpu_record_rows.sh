#!/bin/bash
# Record of the SURVEY 8(f) rows on the current build: LBP bench (both arms)
# with an ncu capture of its kernel, the response-field / sweep bench with an
# ncu capture of the row kernel; summaries as markdown, .ncu-rep dropped.
#   gpu_record_rows.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-r02m}
python bench.py --config c5lbp > gpurun_out/${T}_bench_lbp.json 2> gpurun_out/${T}_bench_lbp.err; echo "lbp rc=$?"
python bench.py --config c5lbp --impl reference > gpurun_out/${T}_bench_lbp_ref.json 2> gpurun_out/${T}_bench_lbp_ref.err; echo "lbp ref rc=$?"
python tools/bench_field.py > gpurun_out/${T}_field_bench.jsonl 2> gpurun_out/${T}_field.err; echo "field rc=$?"
L="python bench.py --config c5lbp --images 16384 --steps 1 --warmup 3 --no-cpu --no-e2e"
$L > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
   -k regex:ldp_fast_kernelILi0ELi2ELb1ELb1ELb1ELb0ELi5E -s 3 -c 1 -o gpurun_out/${T}_lbp $L > gpurun_out/${T}_lbp_ncu.log 2>&1; echo "lbp ncu rc=$?"
F="python tools/bench_field.py --images 512 --steps 2 --warmup 1"
$F > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:response_field_row -s 2 -c 1 \
   -o gpurun_out/${T}_field $F > gpurun_out/${T}_field_ncu.log 2>&1; echo "field ncu rc=$?"
for r in lbp field; do
  [ -f gpurun_out/${T}_$r.ncu-rep ] || continue
  python tools/ncu_summary.py gpurun_out/${T}_$r.ncu-rep gpurun_out/${T}_ncu_${r}_kernel.md > /dev/null 2>&1
  python tools/ncu_brief.py gpurun_out/${T}_$r.ncu-rep > gpurun_out/${T}_ncu_${r}.txt 2>&1
  rm -f gpurun_out/${T}_$r.ncu-rep
done
cat gpurun_out/${T}_field_bench.jsonl | cut -c1-300
