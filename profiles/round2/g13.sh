mkdir -p gpurun_out
T=g13
VARIANTS="cur2 best_nrc_acs" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
TSB200_LIB=$PWD/build_variants/lib_rftrace.so timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_rf_trace.log 2>&1; echo trace rc $?
