#!/bin/bash
# One gpurun pass: smoke, a pytest selection, the default bench line (and optional extras).
#   TAG=name [KEXPR="pytest -k expression"] [FILES="tests/x.py ..."] [BENCH=1] [BENCHARGS=...] tools/gpu_round.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
if [ -n "$KEXPR$FILES" ]; then
  if [ -n "$KEXPR" ]; then
    timeout ${PYT_TIMEOUT:-1800} python -m pytest ${FILES:-tests} -q -m gpu -x -k "$KEXPR" > gpurun_out/${TAG}_pytest.log 2>&1
  else
    timeout ${PYT_TIMEOUT:-1800} python -m pytest ${FILES:-tests} -q -m gpu -x > gpurun_out/${TAG}_pytest.log 2>&1
  fi
  tail -${PYT_TAIL:-6} gpurun_out/${TAG}_pytest.log
fi
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py --no-cpu-baseline $BENCHARGS > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  cut -c1-600 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
fi
