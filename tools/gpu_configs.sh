#!/bin/bash
# Bench lines of every BASELINE config (both arms), one JSON line each, into
# gpurun_out/${TAG}_configs.jsonl (C3 for k = 1, 3, 5).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01h}
OUT=gpurun_out/${TAG}_configs.jsonl
: > $OUT
for a in "--config c1" "--config c2" "--config c3 --k 1" "--config c3 --k 3" "--config c3 --k 5" "--config c4"; do
  timeout 600 python bench.py $a >> $OUT 2>> gpurun_out/${TAG}_configs.err; echo "b200 $a rc=$?"
  timeout 600 python bench.py $a --impl reference >> $OUT 2>> gpurun_out/${TAG}_configs.err; echo "ref $a rc=$?"
done
python - "$OUT" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(d.get("impl", "b200"), d["config"]["workload"][:40], d.get("config", {}).get("k"), d["value"],
          d.get("roofline", {}).get("frac"), d.get("e2e", {}).get("value"))
PY
