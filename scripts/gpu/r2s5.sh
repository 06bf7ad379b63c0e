# deferred fold: rates per temperature window + ncu of the lazy kernel (high and low T)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/lazy_rates.py > gpurun_out/s5_rates_f32.jsonl 2>&1; echo rates=$?
timeout 600 python scripts/lazy_rates.py --precision f64 > gpurun_out/s5_rates_f64.jsonl 2>&1; echo rates64=$?
timeout 300 python scripts/lazy_rates.py --n 500 > gpurun_out/s5_rates_n500.jsonl 2>&1; echo rates500=$?
cat gpurun_out/s5_rates*.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s5_lazy_hiT -f python scripts/profile_engine.py --tmin 905 --launches 1 > gpurun_out/s5_ncu1.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s5_lazy_loT -f python scripts/profile_engine.py --t0 0.1 --tmin 0.0905 --launches 1 > gpurun_out/s5_ncu2.log 2>&1; echo ncu2=$?
