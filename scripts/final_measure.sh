#!/bin/bash
# Round-end measurement (under gpurun): bench lines of both arms, the ncu
# launch list of the bench command, and one --set full capture of the top
# kernels of one steady frame (profile_frame.py: the third composited frame's
# 12 matching launches, after the second's). Usage: bash scripts/final_measure.sh TAG   (e.g. r02c)
TAG=${1:-r02c}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_line.json 2> gpurun_out/${TAG}_bench.err
echo "== ours"; tail -1 gpurun_out/${TAG}_bench_line.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_reference_line.json \
    2> gpurun_out/${TAG}_bench_reference.err
echo "== reference"; tail -1 gpurun_out/${TAG}_bench_reference_line.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${TAG}_ncu_launches.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt
echo "== launches"; head -12 gpurun_out/${TAG}_launch_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_pcg_tmem|k_agg_tma2|k_cost_slices|k_wta_slices|k_flow_patch_w|k_ref_slow|k_agg_fix_out" \
    -s 12 -c 12 -o gpurun_out/${TAG}_full python scripts/profile_frame.py 5 \
    > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "== full"; tail -2 gpurun_out/${TAG}_ncu_full.log
