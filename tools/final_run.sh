#!/bin/bash
# One GPU call's evidence for a commit (run under gpurun from the repo root):
# the GPU suite, smoke(), the bench line and the reference arm, the launch
# list, the L2 reduction counters (fp64 and deterministic modes) and a
# --set full capture of the step kernels, all into gpurun_out/<tag>_*.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/final_run.sh r2f'
# Summaries: tools/launch_summary.py, ncu_summary.py, ncu_atomics.py,
# ncu_traffic.py (profiles/README.md).
set -x
T=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/${T}_ncu_launch.log 2>&1
M=$(python -c "import tools.ncu_atomics as n; print(','.join(n.METRICS))")
ncu --metrics $M --clock-control none -k regex:"k_g2p2g_gel|k_grid_update_boxes|k_ind_cols|k_p2g_gel_tile|k_finalize" -s 30 -c 12 -o gpurun_out/${T}_red python tools/profile_run.py config2a 3 > gpurun_out/${T}_red.log 2>&1
ncu --metrics $M --clock-control none -k regex:"k_g2p2g_gel|k_grid_update_boxes|k_p2g_gel_tile" -s 30 -c 8 -o gpurun_out/${T}_red_det python tools/profile_run.py config2a-det 3 > gpurun_out/${T}_red_det.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_g2p2g_gel|k_grid_update_boxes|k_finalize|k_capture|k_ind_cols" -s 30 -c 8 -o gpurun_out/${T}_prof python tools/profile_run.py config2a 3 > gpurun_out/${T}_prof.log 2>&1
ls gpurun_out/ | grep "^${T}_"
