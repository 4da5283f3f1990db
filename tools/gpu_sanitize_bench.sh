mkdir -p gpurun_out/r16
python -c "import paper_2409_08729_b200._build as b; b.build()" > gpurun_out/r16/build.log 2>&1
: > gpurun_out/r16/sanitizer.txt
for t in memcheck racecheck synccheck initcheck; do
  echo "== compute-sanitizer --tool $t python tools/sanitize_run.py (U bins 6/8/10/13, SMEM log table)" >> gpurun_out/r16/sanitizer.txt
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py 2>&1 | grep -E "SUMMARY|Error|error|hazard" | head -20 >> gpurun_out/r16/sanitizer.txt
done
bash tools/gpu_round.sh r16 bench
