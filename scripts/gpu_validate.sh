#!/bin/bash
# Round-end validation on one B200: GPU tests, smoke, default bench, launch list of the bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/val_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/val_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/val_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/val_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-decode > /dev/null 2>&1
tail -3 gpurun_out/val_tests.log; cat gpurun_out/val_smoke.log | tail -2; cat gpurun_out/val_bench.json
