python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for rep in 1 2 3; do timeout 300 python tools/probe_c5.py C5; done
timeout 300 python tools/probe_c5.py C4
