#!/bin/bash
# f3 pass: host-raw tests + raw-host benches (C5, then C4 if the box has the RAM)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
free -g > gpurun_out/f3_mem.txt; nproc >> gpurun_out/f3_mem.txt
timeout 900 python -m pytest tests/test_gpu_f3.py -q -x --durations=10 > gpurun_out/pytest_f3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f3.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --raw-host --no-cpu --no-b1 > gpurun_out/bench_c5_rawhost.json 2> gpurun_out/bench_c5_rawhost.log
avail=$(free -g | awk '/Mem:/{print $7}')
if [ "$avail" -gt 260 ]; then
  timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --raw-host --no-cpu --no-b1 > gpurun_out/bench_c4_rawhost.json 2> gpurun_out/bench_c4_rawhost.log
fi
exit 0
