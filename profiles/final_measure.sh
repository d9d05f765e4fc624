# usage: final_measure.sh TAG -- default bench line, step timeline, k_update
# ncu (full + warm application replay), launch list of the default command
T=$1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo bench rc $?
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo ref rc $?
TSB200_LIB=$PWD/build_variants/lib_tl.so timeout 600 python profiles/timeline.py > gpurun_out/${T}_timeline.json 2> gpurun_out/${T}_timeline.err; echo tl rc $?
bash profiles/ncu_update.sh ${T}
