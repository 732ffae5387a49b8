python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
RQRCP_PANEL=cqr timeout 300 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/plain.log 2>&1 && \
RQRCP_PANEL=cqr timeout 900 ncu --set full --clock-control none --import-source on -k "regex:cqr_recon|cqr_chol" -s 6 -c 3 -o gpurun_out/r02_cqr -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_cqr.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_cqr.log
