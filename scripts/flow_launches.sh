#!/bin/bash
# Per-level k_flow_patch_w durations (ncu launch list, 3 composited frames)
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_flow_patch --csv \
    --log-file gpurun_out/flowl.csv python scripts/profile_frame.py 3 > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open('gpurun_out/flowl.csv')) if len(r) > 10 and r[0].isdigit()]
print("k_flow_patch (grid, ns):", [(r[8], r[-1]) for r in rows[:5]])
PY
