set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo plain=$?; tail -3 gpurun_out/san_plain.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/memcheck.log 2>&1; echo memcheck=$?; tail -8 gpurun_out/memcheck.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=5 > gpurun_out/pytest_full.log 2>&1; echo full=$?; tail -8 gpurun_out/pytest_full.log
