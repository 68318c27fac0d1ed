#!/bin/bash
# ncu evidence for the bench command (config $CFG): launch list (time only) + one full capture per top kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CFG=${CFG:-4}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu --no-b1"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
$CMD > gpurun_out/ncu_plain_c$CFG.json 2> gpurun_out/ncu_plain_c$CFG.log && [ -z "$NO_LIST" ] && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c$CFG.csv $CMD > gpurun_out/ncu_launch_c$CFG.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch_c$CFG.log
for K in ${KERNELS:-k_lbt k_refine1 k_summarize_tma}; do
  tag=$(echo "$K" | tr -cd 'a-z0-9_')
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-0} -c 1 -o gpurun_out/full_c${CFG}_$tag -f $CMD > gpurun_out/ncu_full_c${CFG}_$tag.log 2>&1
  echo "full $K rc=$?" >> gpurun_out/ncu_full_c${CFG}_$tag.log
done
exit 0
