mkdir -p gpurun_out
T=g19
VARIANTS="cur3 pubhash" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
for v in cur3 pubhash; do for k in 1 2; do python -c "
import json; x=json.load(open('gpurun_out/abv_${v}_$k.json')); print('$v', x['ms_per_step'], x['e2e']['value']/1e9)"; done; done >> gpurun_out/${T}_ab.txt
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_queries.py tests/test_gpu_configs.py --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc $?
