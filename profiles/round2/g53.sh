mkdir -p gpurun_out
timeout 300 python profiles/timeline.py > gpurun_out/g53_tl_if.json 2>/dev/null; echo rc $?
TSB_DEBUG=8 timeout 300 python profiles/timeline.py > gpurun_out/g53_tl_gated.json 2>/dev/null; echo rc $?
for f in if gated; do python -c "
import json; t=json.load(open('gpurun_out/g53_tl_$f.json')); print('$f', t['step_period_us_median'], t['phase_start_us_median'], t['phase_us_median'])"; done
