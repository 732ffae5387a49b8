python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:rq::" -s 150 -c 120 --csv --log-file gpurun_out/r02_c4_panel_launches.csv python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu.log 2>&1; echo ncu=$?
