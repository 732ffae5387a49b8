# Final GPU suite at HEAD (C5 prefix parity to k' = 512 by default) with its total duration.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q --durations=6 > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_gpu_final.log
