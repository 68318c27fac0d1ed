#!/bin/bash
# f3 sweep: raw-host benches with seed counts; C4 raw-host
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for s in 64 256 1024; do
  timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --raw-host --no-cpu --no-b1 --both 0 --index-seeds $s > gpurun_out/bench_c5_rawhost_s$s.json 2> gpurun_out/bench_c5_rawhost_s$s.log
done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --raw-host --no-cpu --no-b1 --both 0 --path flat > gpurun_out/bench_c5_rawhost_flat.json 2> gpurun_out/bench_c5_rawhost_flat.log
for s in 256 1024; do
timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --raw-host --no-cpu --no-b1 --both 0 --index-seeds $s > gpurun_out/bench_c4_rawhost_s$s.json 2> gpurun_out/bench_c4_rawhost_s$s.log
done
free -g >> gpurun_out/bench_c4_rawhost_s1024.log
exit 0
