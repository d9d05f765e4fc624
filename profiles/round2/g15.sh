mkdir -p gpurun_out
T=g15
VARIANTS="cur3 keep" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
VARIANTS="keep cur3" sh profiles/round2/abv.sh > gpurun_out/${T}_ab2.txt 2>&1; echo ab rc $?
