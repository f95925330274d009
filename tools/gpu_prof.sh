#!/bin/bash
# ncu --set full captures of selected conv_tc launches (by index among conv_tc launches) and the stem.
# usage: IDX="18 19" STEM=1 bash tools/gpu_prof.sh
set -u
mkdir -p gpurun_out
for s in ${IDX:-18}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s $s -c 1 \
  -o gpurun_out/prof_tc_$s -f python tools/profile_forward.py --reps 1 > gpurun_out/ncu_tc_$s.log 2>&1; echo "ncu $s rc=$?"
done
if [ "${STEM:-0}" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stem -c 1 \
  -o gpurun_out/prof_stem -f python tools/profile_forward.py --reps 1 > gpurun_out/ncu_stem.log 2>&1; echo "ncu stem rc=$?"
fi
