# one ncu --set full capture of selected kernels (KREGEX) of one warm factorization
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
CFG=${CFG:-C2}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-4} \
  -o gpurun_out/${NAME:-full} -f python tools/profile_step.py --config $CFG > gpurun_out/ncu_full_${NAME:-full}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full_${NAME:-full}.log
