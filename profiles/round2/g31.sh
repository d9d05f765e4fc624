mkdir -p gpurun_out
timeout 600 python profiles/timeline.py > gpurun_out/g31_timeline.json 2> gpurun_out/g31_timeline.err; echo tl rc $?
