mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/reloc_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/reloc_pytest.log
VARIANTS="${VARIANTS:-base reloc}" sh profiles/ab.sh
