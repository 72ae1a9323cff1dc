# Round-2 whole-frame parity evidence for the final kernel (profiles/r2_*parity*.json)
set -u
timeout 1500 python tools/full_frame_parity.py --json gpurun_out/ffp_final.json > gpurun_out/ffp_final.log 2>&1; echo ffp=$?
timeout 1500 python tools/parity_sweep.py --json gpurun_out/sweep_final.json > gpurun_out/sweep_final.log 2>&1; echo sweep=$?
timeout 1500 python tools/parity_sweep.py --wide --json gpurun_out/sweep_wide_final.json > gpurun_out/sweep_wide_final.log 2>&1; echo wide=$?
timeout 900 python tools/scene_parity.py 6 --json gpurun_out/scene_final.json > gpurun_out/scene_final.log 2>&1; echo scene=$?
