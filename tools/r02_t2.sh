set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q --durations=15 > gpurun_out/pytest_parity.log 2>&1; echo parity=$?; tail -45 gpurun_out/pytest_parity.log
