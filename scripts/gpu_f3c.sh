#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2009_00166_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --raw-host --no-cpu --no-b1 --both 0 > gpurun_out/f3c_c4.json 2> gpurun_out/f3c_c4.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --raw-host --no-cpu --no-b1 --both 0 > gpurun_out/f3c_c5.json 2> gpurun_out/f3c_c5.log
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --raw16 --no-cpu --no-b1 --both 0 > gpurun_out/f3c_c2_r16.json 2> gpurun_out/f3c_c2_r16.log
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-b1 --both 0 > gpurun_out/f3c_c2.json 2> gpurun_out/f3c_c2.log
exit 0
