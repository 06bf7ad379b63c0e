cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s8_lazy_hiT -f python scripts/profile_engine.py --tmin 905 --launches 1 > gpurun_out/s8_ncu1.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s8_lazy_loT -f python scripts/profile_engine.py --t0 0.1 --tmin 0.0905 --launches 1 > gpurun_out/s8_ncu2.log 2>&1; echo ncu2=$?
PSA_LIB_PATH=gpu_variants/unroll2/libparsa_b200.so timeout 600 python scripts/lazy_rates.py > gpurun_out/s8_rates_u2.jsonl 2>&1
cat gpurun_out/s8_rates_u2.jsonl | cut -c1-200
