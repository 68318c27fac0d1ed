#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PARIS_DEBUG=1 python -m paper_2009_00166_b200.build --force > gpurun_out/build_dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_parity.py -q -x -k "k or parity" > gpurun_out/pytest_kdbg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_kdbg.log
python -m paper_2009_00166_b200.build --force > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
for c in 5 2; do
timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-b1 --both 0 > gpurun_out/k_c$c.json 2> gpurun_out/k_c$c.log
done
exit 0
