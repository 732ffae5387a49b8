# ncu --set full of the register-grid sample QRCP (S2) and the S5 GEMMs of one C4
# panel at HEAD (v14), raw pages exported on the box.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sample_qrcp_reg" -s 2 -c 1 -o gpurun_out/r02_v14_c4_sq -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_sq.log 2>&1; echo ncu1=$?; tail -2 gpurun_out/ncu_sq.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gemm_upd_ws_kernel|gemm_ws_kernel<4, 4, 4, 2, 32, 4, 1>" -s 12 -c 4 -o gpurun_out/r02_v14_c4_gemm -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_gemm.log 2>&1; echo ncu2=$?; tail -2 gpurun_out/ncu_gemm.log
for r in r02_v14_c4_sq r02_v14_c4_gemm; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null; done
ls -la gpurun_out
# launch list of the bench command (library kernels only: the input generator's cuSOLVER / torch kernels are not the path)
timeout 900 ncu --kernel-name-base demangled -k regex:rq:: --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02_v14_c4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu3=$?
