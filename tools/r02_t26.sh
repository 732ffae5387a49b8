python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "register_grid or sample_qrcp" > gpurun_out/pytest_sq.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_sq.log
RQRCP_TRACE=1 RQRCP_TRACE_PANEL=3 timeout 300 python tools/profile_step.py --config C5 --warm 0 2>&1 | grep -i "sample\|rank"
