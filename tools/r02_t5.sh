python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat tools/dmma_lat.cu && ./tools/dmma_lat > gpurun_out/dmma_lat.json; cat gpurun_out/dmma_lat.json
timeout 300 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_c4.log 2>&1; echo ncu1=$?
RQRCP_PANEL=cqr timeout 300 python tools/profile_step.py --config C4 --warm 0 > gpurun_out/plain_c4cqr.log 2>&1 && \
RQRCP_PANEL=cqr timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4cqr_launches.csv python tools/profile_step.py --config C4 --warm 0 > gpurun_out/ncu_c4cqr.log 2>&1; echo ncu2=$?
tail -2 gpurun_out/plain_c4.log gpurun_out/plain_c4cqr.log
