# ncu --set full of the S5 W = V^T A22 kernel at HEAD (C4, around panel 12)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemm_ws_kernel<.int.4, .int.4, .int.4, .int.2, .int.32, .int.4, .int.1>" -s 36 -c 3 -o gpurun_out/r02_v14_c4_w -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_w.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_w.log
ncu -i gpurun_out/r02_v14_c4_w.ncu-rep --page raw --csv > gpurun_out/r02_v14_c4_w.raw.csv 2>/dev/null
