cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fx_gemm -s 3 -c 1 -o gpurun_out/prof_fx3 python profiles/ab_fx.py build/ab/fx3.so > gpurun_out/ncu_fx3.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_fx3.log
