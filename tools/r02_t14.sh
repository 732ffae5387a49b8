python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?; grep -E "Elapsed|Maximum resident" gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 300 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemm_upd_ws|gemm_tma_kernel<4, 4, 4, 2|panel_qr_kernel|sample_qrcp_reg" -s 12 -c 8 -o gpurun_out/r02_c4_full_v3 -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?; tail -3 gpurun_out/ncu_full.log
