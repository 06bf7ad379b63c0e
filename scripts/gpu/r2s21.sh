cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nm_kernel -c 1 -o gpurun_out/s21_nm -f python scripts/nm_rate.py 20000 > gpurun_out/s21_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/s21_ncu.log
