# One-off: C5 against the prefix oracle to k' = 512 (4 panels; the default test compares 2 to keep the suite short).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
RQRCP_TEST_C5_PANELS=4 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k test_C5_full_size --durations=3 > gpurun_out/pytest_c5_4panels.log 2>&1; echo pytest=$?; tail -8 gpurun_out/pytest_c5_4panels.log
