#!/bin/bash
# One GPU session: targeted tests, the full -m gpu suite, a bench line (no CPU
# baseline) and an ncu launch list of 6 frames. Usage (under gpurun):
#   bash scripts/gpu_check.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:-volumes}
timeout 900 python -m pytest tests/test_gpu_stereo.py -q -x -k "$K" --timeout 600 -p no:cacheprovider > gpurun_out/vol.log 2>&1
echo "== targeted"; tail -3 gpurun_out/vol.log
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/gputests.log 2>&1
echo "== gpu suite"; tail -3 gpurun_out/gputests.log; grep -E "^FAILED|Error" gpurun_out/gputests.log | head -10
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "== bench"; python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), round(d['e2e']['value'],1), d['stage_ms'])" || tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_frame.py 6 > gpurun_out/ncu.log 2>&1
echo "== launches"; python scripts/launch_summary.py gpurun_out/launches.csv | head -16
