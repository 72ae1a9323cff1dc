# Round-2 checks: full GPU suite (hazard report written to gpurun_out/),
# chain diagnosis, bench line with the in-bench parity block.
set -u
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
rm -f gpurun_out/hazards.json
PGG_REPORT_DIR=gpurun_out timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/chain_flips.py 160 120 4 9 --json gpurun_out/chain_160.json > gpurun_out/chain_160.log 2>&1; echo chain=$?
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
