# A/B of hub small table size (BitHash<9> <=512 keys vs BitHash<8> <=256 keys)
for sb in 9 8; do
  BFLY_HUB_SMALL_BITS=$sb python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$sb.json 2>gpurun_out/ab_$sb.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$sb.json'));print($sb, round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items() if k.startswith('hub_')})"
  grep e2e gpurun_out/ab_$sb.err
done
