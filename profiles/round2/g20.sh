mkdir -p gpurun_out
T=g20
VARIANTS="cur3 pubwarp" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
for v in cur3 pubwarp; do for k in 1 2; do python -c "
import json; x=json.load(open('gpurun_out/abv_${v}_$k.json')); print('$v', x['ms_per_step'], x['e2e']['value']/1e9)"; done; done >> gpurun_out/${T}_ab.txt
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_golden.py tests/test_gpu_queries.py --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
