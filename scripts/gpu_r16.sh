#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2009_00166_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_f3.py -q -x > gpurun_out/pytest_r16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r16.log
for c in 4 2 5; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-b1 --both 0 --raw16 > gpurun_out/r16_c$c.json 2> gpurun_out/r16_c$c.log
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-b1 --both 0 > gpurun_out/r32_c$c.json 2> gpurun_out/r32_c$c.log
done
exit 0
