# deferred-fold kernel: GPU parity suite + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -k "not c3_full and not c4_hybrid_table8" > gpurun_out/s3_pytest.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/s3_pytest.log
timeout 600 python bench.py --no-configs --no-companion > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s3_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d.get('parity'))" 
tail -5 gpurun_out/s3_bench.err
