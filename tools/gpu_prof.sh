# launch list of one warm factorization (ncu, serialised, cold-ish caches)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
CFG=${CFG:-C2}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv python tools/profile_step.py --config $CFG > gpurun_out/ncu_${CFG}.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_${CFG}.csv --last ${LAST:-200}
