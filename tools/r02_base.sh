# Round-2 baseline at C4 (current code): plain run, then ncu --set full of the
# S5 GEMMs, the grid panel kernel and the register-grid sample QRCP at C4.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/r02_base_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:gemm_upd_tma|gemm_tma_kernel|panel_qr_kernel|sample_qrcp_reg" -s 8 -c 8 -o gpurun_out/r02_c4_full -f python tools/profile_step.py --config C4 --warm 0 > gpurun_out/r02_c4_ncu.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/r02_c4_ncu.log
