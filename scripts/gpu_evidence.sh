#!/bin/bash
# Round evidence: default bench (C4) + all configs + ncu launch list of the default command + full captures
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ev/smoke.log
timeout 900 python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.log
for c in 1 2 3 5; do timeout 900 python bench.py --config $c > gpurun_out/ev/bench_c$c.json 2> gpurun_out/ev/bench_c$c.log; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-b1 --both 0"
$CMD > gpurun_out/ev/ncu_plain.json 2> gpurun_out/ev/ncu_plain.log && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ev/launches_c4.csv $CMD > gpurun_out/ev/ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/ev/ncu_launch.log
ncu --set full --clock-control none --import-source on -k regex:k_lbi -s 1 -c 1 -o gpurun_out/ev/full_c4_k_lbi -f $CMD > gpurun_out/ev/ncu_full_lbi.log 2>&1; echo "rc=$?" >> gpurun_out/ev/ncu_full_lbi.log
ncu --set full --clock-control none --import-source on -k regex:k_refine1u -s 3 -c 1 -o gpurun_out/ev/full_c4_k_refine1 -f $CMD > gpurun_out/ev/ncu_full_ref.log 2>&1; echo "rc=$?" >> gpurun_out/ev/ncu_full_ref.log
ncu --set full --clock-control none --import-source on -k regex:k_summarize_seg -s 1 -c 1 -o gpurun_out/ev/full_c4_k_summarize -f $CMD > gpurun_out/ev/ncu_full_sum.log 2>&1; echo "rc=$?" >> gpurun_out/ev/ncu_full_sum.log
ncu --set full --clock-control none --import-source on -k regex:k_blkmask -s 1 -c 1 -o gpurun_out/ev/full_c4_k_blkmask -f $CMD > gpurun_out/ev/ncu_full_blk.log 2>&1; echo "rc=$?" >> gpurun_out/ev/ncu_full_blk.log
CMDF="python bench.py --steps 2 --warmup 3 --no-cpu --no-b1 --both 0 --path flat"
ncu --set full --clock-control none --import-source on -k regex:k_lbt -s 1 -c 1 -o gpurun_out/ev/full_c4_k_lbt -f $CMDF > gpurun_out/ev/ncu_full_lbt.log 2>&1; echo "rc=$?" >> gpurun_out/ev/ncu_full_lbt.log
# summaries on the box; keep only the k_lbi report (gpurun copies back <= 64 MiB)
for k in k_lbi k_refine1 k_summarize k_blkmask k_lbt; do
  python scripts/ncu_summary.py gpurun_out/ev/full_c4_$k.ncu-rep > gpurun_out/ev/full_c4_${k}_summary.txt 2>&1
done
python scripts/ncu_hot.py gpurun_out/ev/full_c4_k_lbi.ncu-rep k_lbi 30 > gpurun_out/ev/full_c4_k_lbi_hot_sass.txt 2>&1
python scripts/launch_shares.py gpurun_out/ev/launches_c4.csv > gpurun_out/ev/launches_c4_shares.txt 2>&1
rm -f gpurun_out/ev/full_c4_k_refine1.ncu-rep gpurun_out/ev/full_c4_k_summarize.ncu-rep gpurun_out/ev/full_c4_k_blkmask.ncu-rep gpurun_out/ev/full_c4_k_lbt.ncu-rep
exit 0
