#!/bin/bash
# One GPU-box session: GPU tests, the bench line, and (optionally) the CPU model check.
#   bash tools/box/round.sh TAG [tests|bench|cpucheck ...]
TAG=$1; shift
mkdir -p gpurun_out
for step in "$@"; do
  case $step in
    tests) python -m pytest tests -m gpu -q -s > gpurun_out/${TAG}_gputests.log 2>&1
           echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_gputests.log ;;
    bench) python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
           echo "bench rc=$?"; tail -c 600 gpurun_out/${TAG}_bench.json ;;
    cpucheck) python tools/cpu_model_check.py 0 1 > gpurun_out/${TAG}_cpucheck.log 2>&1
           echo "cpucheck rc=$?"; tail -4 gpurun_out/${TAG}_cpucheck.log; cp profiles/r2_cpu_model_check_*.json gpurun_out/ 2>/dev/null ;;
  esac
done
