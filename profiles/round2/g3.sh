# k_update variant A/B (block-compacted MOBIL sides vs original; occupancy) + query timing
mkdir -p gpurun_out
VARIANTS="orig compact compact_m5 compact_128x8 orig_m5" sh profiles/round2/abv.sh > gpurun_out/g3_ab.txt 2>&1; echo ab rc $?
timeout 900 python -m pytest -q -m gpu tests/test_gpu_queries.py -x --timeout 600 -s > gpurun_out/g3_pytest.log 2>&1; echo pytest rc $?
