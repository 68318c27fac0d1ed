#!/bin/bash
# Round-2 evidence (final: with the tensor-core filter k_gf on the flat path): build as the driver does, all GPU tests (incl. full size), smoke, the ncu
# launch list of the default command and full captures of the top kernels (summaries + DRAM
# traffic JSON, copied to profiles/ncu_traffic.json so the bench lines below report
# roofline.traffic of this very build), then the default bench line, every config, the
# reference arm and torchrun N=1 (sharded path).  OUT=gpurun_out/<tag>
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/ev6}
mkdir -p $OUT
(free -g; nproc; lscpu | grep -i "model name"; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv) > $OUT/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
sha256sum paper_2009_00166_b200/libparis.so > $OUT/lib_sha.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
if [ -z "$SKIP_TESTS" ]; then
  timeout 3000 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
fi
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-b1 --both 0 --no-sweep"
$CMD > $OUT/ncu_plain.json 2> $OUT/ncu_plain.log && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "rc=$?" >> $OUT/ncu_launch.log
python scripts/launch_shares.py $OUT/launches_c4.csv > $OUT/launches_c4_shares.txt 2>&1
for spec in "k_lbi 1 1" "k_refine1m 2 2" "k_summarize_seg 1 1" "k_blkmask 1 1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -o $OUT/full_c4_$1 -f $CMD > $OUT/ncu_full_$1.log 2>&1
  python scripts/ncu_summary.py $OUT/full_c4_$1.ncu-rep > $OUT/full_c4_$1_summary.txt 2>&1
  python scripts/ncu_hot.py $OUT/full_c4_$1.ncu-rep $1 40 > $OUT/full_c4_$1_hot_sass.txt 2>&1
done
CMDF="python bench.py --steps 2 --warmup 3 --no-cpu --both 0 --no-sweep --path flat"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lb1t -s 1 -c 1 -o $OUT/full_c4_k_lb1t -f $CMDF > $OUT/ncu_full_k_lb1t.log 2>&1
python scripts/ncu_summary.py $OUT/full_c4_k_lb1t.ncu-rep > $OUT/full_c4_k_lb1t_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k k_gf -s 1 -c 1 -o $OUT/full_c4_k_gf -f $CMDF > $OUT/ncu_full_k_gf.log 2>&1
python scripts/ncu_summary.py $OUT/full_c4_k_gf.ncu-rep > $OUT/full_c4_k_gf_summary.txt 2>&1
python scripts/ncu_hot.py $OUT/full_c4_k_gf.ncu-rep k_gf 40 > $OUT/full_c4_k_gf_hot_sass.txt 2>&1
python scripts/ncu_traffic.py $OUT > $OUT/ncu_traffic.json 2> $OUT/ncu_traffic.log && cp $OUT/ncu_traffic.json profiles/ncu_traffic.json
rm -f $OUT/full_c4_k_refine1m.ncu-rep $OUT/full_c4_k_summarize_seg.ncu-rep $OUT/full_c4_k_blkmask.ncu-rep $OUT/full_c4_k_lb1t.ncu-rep $OUT/full_c4_k_gf.ncu-rep
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.log
for c in 1 2 3 5; do timeout 900 python bench.py --config $c > $OUT/bench_c$c.json 2> $OUT/bench_c$c.log; done
# the tensor-core filter on the index path too (variant key 3 = 1) and off everywhere (= 0): A/B lines
for c in 4 3 5; do
  PARIS_VARIANT="3=1" timeout 900 python bench.py --config $c --no-cpu --no-b1 --both 0 > $OUT/bench_c${c}_gfindex.json 2> $OUT/bench_c${c}_gfindex.log
  PARIS_VARIANT="3=0" timeout 900 python bench.py --config $c --no-cpu --no-b1 --both 0 --path flat > $OUT/bench_c${c}_flat_nogf.json 2> $OUT/bench_c${c}_flat_nogf.log
  timeout 900 python bench.py --config $c --no-cpu --no-b1 --both 0 --path flat > $OUT/bench_c${c}_flat_gf.json 2> $OUT/bench_c${c}_flat_gf.log
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > $OUT/bench_torchrun1.json 2> $OUT/bench_torchrun1.log
python scripts/bench_brief.py $OUT/bench_*.json > $OUT/brief.txt 2>&1
exit 0
