#!/bin/bash
# build, gpu tests, smoke, benches ($CONFIGS), then an ncu capture of the LB/summarize/refine kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
for c in $CONFIGS; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 $BENCH_ARGS > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.log
done
if [ -n "$PROF" ]; then
  python scripts/prof_lb.py > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$PROF" -c ${PROF_C:-6} -o gpurun_out/prof -f python scripts/prof_lb.py > gpurun_out/prof_ncu.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/prof_ncu.log
fi
exit 0
