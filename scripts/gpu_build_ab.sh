#!/bin/bash
# A/B of compile-time tuning flags: for each flag set (";"-separated; "-" = defaults) build with
# those flags and run scripts/ab_variants.py with the given args at each config; the default
# build is restored at the end.  OUT=gpurun_out/<tag> SETS="-;PARIS_REFM_KP=2" CONFIGS="4 3"
# ABARGS="--key 2 --values 1 --reps 3"
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/bab}
mkdir -p $OUT
IFS=';' read -ra SETL <<< "${SETS:--}"
for fs in "${SETL[@]}"; do
  if [ "$fs" = "-" ]; then envs=""; else envs="$fs"; fi
  env $envs python -m paper_2009_00166_b200.build --force > "$OUT/build_${fs//[ =]/_}.log" 2>&1 || { echo "build $fs failed"; continue; }
  for c in ${CONFIGS:-4}; do
    echo "{\"flags\": \"$fs\", \"config\": $c}" >> $OUT/ab.jsonl
    timeout 900 python scripts/ab_variants.py --config $c ${ABARGS} >> $OUT/ab.jsonl 2>> $OUT/ab_err.log
  done
done
python -m paper_2009_00166_b200.build --force > $OUT/build_restore.log 2>&1
cat $OUT/ab.jsonl
exit 0
