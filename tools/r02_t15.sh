python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
start=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$? wall=$(( $(date +%s) - start ))s; tail -2 gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
start=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$? wall=$(( $(date +%s) - start ))s; tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 300 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gemm_tma_kernel|gemm_upd_ws" -s 6 -c 3 -o gpurun_out/r02_c4_gemm_v3 -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_full.log
