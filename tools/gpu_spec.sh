python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_spec.py -q > gpurun_out/pytest_spec.log 2>&1; echo spec=$?
