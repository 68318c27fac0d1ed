#!/bin/bash
# ncu full captures of one kernel under two variant settings (PARIS_VARIANT), C4 bench command.
# OUT=gpurun_out/<tag> K=k_refine1q VA="2=0" VB="2=1" SKIP=2
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/ncuv}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-b1 --both 0 --no-sweep ${NCU_ARGS}"
for tag in A B; do
  if [ $tag = A ]; then V=$VA; else V=$VB; fi
  PARIS_VARIANT=$V timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-1} -c 1 -o $OUT/full_${K}_$tag -f $CMD > $OUT/ncu_$tag.log 2>&1
  python scripts/ncu_summary.py $OUT/full_${K}_$tag.ncu-rep > $OUT/full_${K}_${tag}_summary.txt 2>&1
  python scripts/ncu_hot.py $OUT/full_${K}_$tag.ncu-rep $K 40 > $OUT/full_${K}_${tag}_hot_sass.txt 2>&1
done
exit 0
