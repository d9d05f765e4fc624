mkdir -p gpurun_out
timeout 600 python profiles/round2/e2e_step_overhead.py > gpurun_out/g46_e2e.json 2> gpurun_out/g46_e2e.err; echo rc $?
cat gpurun_out/g46_e2e.json; tail -3 gpurun_out/g46_e2e.err
