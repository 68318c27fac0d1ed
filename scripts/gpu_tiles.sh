cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PARIS_DEBUG_TILES=1 timeout 600 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu --no-b1 --both 0 > gpurun_out/tiles.json 2> gpurun_out/tiles.log
PARIS_DEBUG_TILES=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-b1 --both 0 > gpurun_out/tiles5.json 2> gpurun_out/tiles5.log
