mkdir -p gpurun_out
timeout 3300 python tools/long_parity.py 200 3 > gpurun_out/g37_long_parity.log 2>&1; echo long rc $?
