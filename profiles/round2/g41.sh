mkdir -p gpurun_out
VARIANTS="base14 pf48 pf32" sh profiles/round2/abv.sh > gpurun_out/g41_ab.txt 2>&1; echo ab rc $?
