#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2009_00166_b200.build --force > gpurun_out/build.log 2>&1
for s in 1024 2048 4096; do
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-b1 --both 0 --index-seeds $s > gpurun_out/seeds_$s.json 2> gpurun_out/seeds_$s.log
done
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-b1 --both 0 > gpurun_out/seeds_c3.json 2> gpurun_out/seeds_c3.log
exit 0
