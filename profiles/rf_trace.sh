# resolve fast-path phase timing (globaltimer printf variant)
mkdir -p gpurun_out
TSB200_LIB=$PWD/build_variants/lib_rftrace.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rf_trace.log 2>&1; echo trace rc $?
