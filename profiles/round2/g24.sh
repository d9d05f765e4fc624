mkdir -p gpurun_out
T=g24
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc $?
timeout 3000 python -m pytest -q -m gpu tests --timeout 1200 --durations=15 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
