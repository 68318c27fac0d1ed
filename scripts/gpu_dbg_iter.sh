#!/bin/bash
# debug-checked build (device bounds checks) on the index tests, then the release iteration
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PARIS_DEBUG=1 python -m paper_2009_00166_b200.build --force > gpurun_out/build_dbg.log 2>&1
timeout 600 python -m pytest tests/test_gpu_index.py -q -x > gpurun_out/pytest_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dbg.log
bash scripts/gpu_iter.sh
