#!/bin/bash
# One gpurun call of the round's checks: host facts, the GPU tests, the bench line (native arm) and
# the reference arm. Usage (from this container): gpurun -- 'bash tools/gpu_check.sh <tag> [pytest args]'
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-chk}; shift
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi -L) > gpurun_out/${T}_host.txt 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider "$@" > gpurun_out/${T}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
fi
if [ "${SKIP_BENCH:-0}" != 1 ]; then
  timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/${T}_bench.log 2>&1
  echo "bench rc=$?" >> gpurun_out/${T}_bench.log
fi
if [ "${SKIP_REF:-0}" != 1 ]; then
  timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.log 2>&1
  echo "ref rc=$?" >> gpurun_out/${T}_ref.log
fi
