# A/B: alternate variants to average out box noise
for rep in 1 2; do for v in $VARIANTS; do
  TSB200_LIB=$PWD/build_variants/lib_$v.so timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/ab_${v}_$rep.log 2>&1
done; done
for v in $VARIANTS; do python -c "
import json
r=[json.load(open('gpurun_out/ab_${v}_%d.log'%k)) for k in (1,2)]
print('$v', [round(x['ms_per_step'],4) for x in r], [round(x['config']['pow']['value_pow_glibc']/1e9,3) for x in r])"; done
