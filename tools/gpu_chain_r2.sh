# Round-2 16-frame trajectory evidence for the final kernel (profiles/r2_chain_1080p_16f*.json)
set -u
timeout 1500 python tools/chain_1080p.py 16 --json gpurun_out/chain_final.json > gpurun_out/chain_final.log 2>&1; echo chain=$?
timeout 2400 python tools/chain_1080p.py 16 --ulp --every --json gpurun_out/chain_final_ulp.json > gpurun_out/chain_final_ulp.log 2>&1; echo chain_ulp=$?
