#!/bin/bash
# compute-sanitizer over every kernel (tools/sanitize_run.py), then one bench run.
# usage (from the repo root, under gpurun): bash tools/gpu_sanitize_bench.sh [tag] [note] [nobench]
TAG=${1:-r16}
NOTE=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import paper_2409_08729_b200._build as b; b.build()" > $OUT/build.log 2>&1
: > $OUT/sanitizer.txt
for t in memcheck racecheck synccheck initcheck; do
  echo "== compute-sanitizer --tool $t python tools/sanitize_run.py $NOTE" >> $OUT/sanitizer.txt
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py 2>&1 | grep -E "SUMMARY|Error|error|hazard" | head -20 >> $OUT/sanitizer.txt
done
[ "${3:-}" = "nobench" ] || bash tools/gpu_round.sh $TAG bench
