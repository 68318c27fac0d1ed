#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2009_00166_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_f3.py tests/test_gpu_index.py -q -x > gpurun_out/pytest_f3d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f3d.log
timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --raw-host --no-cpu --no-b1 --both 0 > gpurun_out/f3d_c4.json 2> gpurun_out/f3d_c4.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --raw-host --no-cpu --no-b1 --both 0 > gpurun_out/f3d_c5.json 2> gpurun_out/f3d_c5.log
exit 0
