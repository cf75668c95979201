export BFLY_AGG_CONCURRENT=0
show() { python3 -c "
import json,sys
d=json.load(open('gpurun_out/ab_$1.json'))
print('$1', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k in ('count_phase','hub_small','hub_medium','hub_medium_wide','hub_heavy')})
"; }
tools/ab_env.sh "base=-" "wb512=BFLY_HUB_WIDE_BLOCK=512" "sp2k=BFLY_HUB_SPLIT_UNITS=2048" "sp8k=BFLY_HUB_SPLIT_UNITS=8192" > /dev/null
for n in base wb512 sp2k sp8k; do show $n; done
tools/ab.sh "l1024=-DBFLY_HUB_LIM2=1024 -DBFLY_HUB_SB_BITS=9" > /dev/null
show l1024
