# A/B over (variant lib, bench debug flags) pairs: VARIANTS="lib:debug ..."
mkdir -p gpurun_out
for rep in 1 2; do for vd in $VARIANTS; do v=${vd%%:*}; d=${vd##*:}
  TSB200_LIB=$PWD/build_variants/lib_$v.so timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --debug $d > gpurun_out/ab_${v}_${d}_$rep.log 2>&1
done; done
for vd in $VARIANTS; do v=${vd%%:*}; d=${vd##*:}; python -c "
import json
r=[json.loads(open('gpurun_out/ab_${v}_${d}_%d.log'%k).read().strip().splitlines()[-1]) for k in (1,2)]
print('$v debug $d', [round(x['ms_per_step'],4) for x in r], [round(x['config']['pow']['value_pow_glibc']/1e9,3) for x in r])"; done
