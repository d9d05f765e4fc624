mkdir -p gpurun_out
T=g12
VARIANTS="best best_nrc" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
VARIANTS="best_nrc best" sh profiles/round2/abv.sh > gpurun_out/${T}_ab2.txt 2>&1; echo ab rc $?
