mkdir -p gpurun_out
for k in 1 2; do timeout 300 python profiles/timeline.py > gpurun_out/g44_tl_$k.json 2> gpurun_out/g44_tl_$k.err; echo tl rc $?; done
cat gpurun_out/g44_tl_1.json gpurun_out/g44_tl_2.json
