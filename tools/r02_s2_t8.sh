python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:cqr_" -s 16 -c 8 -o gpurun_out/r02_c4_cqr -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_cqr.log 2>&1; echo ncu1=$?; tail -2 gpurun_out/ncu_cqr.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sample_qrcp_reg" -s 2 -c 1 -o gpurun_out/r02_c4_sq -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_sq.log 2>&1; echo ncu2=$?; tail -2 gpurun_out/ncu_sq.log
