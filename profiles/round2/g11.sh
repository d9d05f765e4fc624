mkdir -p gpurun_out
T=g11
VARIANTS="best best_lin16 best_lin8 best_lx4" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
