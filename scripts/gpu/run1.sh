# GPU session 1 (round 2): GPU tests + C4 SA variants + ncu of the C4 SA kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "not c3_full and not c4_hybrid" > gpurun_out/r1_pytest.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/r1_pytest.log
timeout 300 python scripts/measure_configs.py --only C4 > gpurun_out/r1_c4.jsonl 2>&1; echo c4=$?
PSA_V2_MODE=pair timeout 300 python scripts/measure_configs.py --only C4 > gpurun_out/r1_c4_pair.jsonl 2>&1; echo c4pair=$?
PSA_FORCE_HBM_ROWS=1 timeout 300 python scripts/measure_configs.py --only C4 > gpurun_out/r1_c4_hbm.jsonl 2>&1; echo c4hbm=$?
cat gpurun_out/r1_c4*.jsonl
for P in f32 f64; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_ -c 1 -o gpurun_out/r1_c4_$P -f python scripts/profile_engine.py --n 500 --tmin 989 --precision $P --launches 1 > gpurun_out/r1_ncu_c4_$P.log 2>&1; echo ncu_$P=$?
done
