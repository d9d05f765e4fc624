mkdir -p gpurun_out
T=g16
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc $?
TSB200_LIB=$PWD/build_variants/lib_cur3.so timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_nopub.json 2> gpurun_out/${T}_bench_nopub.err; echo bench rc $?
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench2.json 2> gpurun_out/${T}_bench2.err; echo bench rc $?
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_queries.py tests/test_gpu_configs.py --timeout 900 -x > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc $?
