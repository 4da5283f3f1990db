#!/bin/bash
# One GPU session: build check, FP64 peak, parity tests, smoke, bench, ncu.
# usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag] [what...]
set -u
TAG=${1:-r01}
shift || true
WHAT=${*:-"peak tests smoke bench launches full"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
python -c "import paper_2409_08729_b200._build as b; b.build(); import oracle; oracle.build()" > $OUT/build.log 2>&1
for w in $WHAT; do
  case $w in
    peak)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && timeout 120 /tmp/fp64_peak > $OUT/fp64_peak.json 2>&1 ;;
    tests)
      timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log ;;
    testsall)
      timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log ;;
    bench)
      timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
        python bench.py --steps 2 --warmup 1 --skip-e2e --skip-cpu-baseline --skip-extra > $OUT/launches_bench.log 2>&1 ;;
    methods)
      timeout 600 python tools/method_bench.py > $OUT/methods.json 2> $OUT/methods.err ;;
    full)
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bessel_eval_kernel -s 1 -c 3 \
        -o $OUT/prof -f python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu-baseline --skip-extra --n-per-v 2000000 > $OUT/ncu_full.log 2>&1 ;;
  esac
done
ls -la $OUT
