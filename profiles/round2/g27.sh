mkdir -p gpurun_out
VARIANTS="cur5 l1max l1half" sh profiles/round2/abv.sh > gpurun_out/g27_ab.txt 2>&1; echo ab rc $?
