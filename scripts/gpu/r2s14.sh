cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s14_lazy_hiT -f python scripts/profile_engine.py --tmin 905 --launches 1 > gpurun_out/s14_ncu1.log 2>&1; echo ncu1=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s14_launches.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline --no-companion > gpurun_out/s14_b_ncu.log 2>&1; echo ncul=$?
timeout 900 python bench.py > gpurun_out/s14_bench.json 2> gpurun_out/s14_bench.err; echo bench_rc=$?
ls -la gpurun_out
