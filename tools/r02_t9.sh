python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
RQRCP_SCHEDULE=0 RQRCP_TRACE=1 RQRCP_TRACE_PANEL=3 timeout 300 python tools/profile_step.py --config C4 --warm 0 2>&1 | grep trace
RQRCP_SCHEDULE=0 timeout 300 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/plain.log 2>&1 && \
RQRCP_SCHEDULE=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:rq::|iota" -s 120 -c 80 --csv --log-file gpurun_out/r02_c4_panel_launches.csv python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu.log 2>&1; echo ncu=$?
