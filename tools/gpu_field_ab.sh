#!/bin/bash
# A/B of response-field row-kernel variants (tools/variants/lib_b<band>_c<cols>.so)
for lib in tools/variants/lib_*.so; do
  echo "== $lib"
  ALDP_LIB=$lib python tools/bench_field.py --steps 5 | head -c 300; echo
done
