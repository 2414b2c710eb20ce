#!/bin/bash
# iteration run: full GPU suite on the in-tree library, the parity/fuzz files
# against the variant TESTLIB (changed arithmetic), then interleaved A/B.
#   TESTLIB=variants/libaldp_X.so CFGS="..." gpu_iter2.sh LIB...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest default rc=$?"
tail -2 gpurun_out/pytest_gpu.log
fi
if [ -n "$TESTLIB" ]; then
ALDP_LIB=$TESTLIB timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_properties_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_variant.log 2>&1; echo "pytest $TESTLIB rc=$?"
tail -2 gpurun_out/pytest_variant.log
fi
tools/gpu_ab2.sh "$@"
