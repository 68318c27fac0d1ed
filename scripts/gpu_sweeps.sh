#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2009_00166_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_abi.py -q -x > gpurun_out/pytest_abi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_abi.log
for c in 2 5 4; do
timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-b1 > gpurun_out/sw_c$c.json 2> gpurun_out/sw_c$c.log
done
exit 0
