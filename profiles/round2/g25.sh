mkdir -p gpurun_out
T=g25
VARIANTS="cur4 lx32b10 lx32b8" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
