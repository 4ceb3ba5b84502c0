B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-size-curve --no-check"
run() { tag=$1; shift; env "$@" timeout 300 $B > gpurun_out/r4f_$tag.log 2>&1; python3 - gpurun_out/r4f_$tag.log <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
ps=d['phase_ms_serial']; pp=d['phase_ms']
ser=sum(ps[k] for k in ['baby','mac','rescale','giant','fold'])
print(sys.argv[1].split('_')[-1], 'q/s %.1f step %.2f serial-sum %.2f mac %.2f | pipelined phases'%(d['value'],d['ms_per_step'],ser,ps['mac']), {k:round(v,2) for k,v in pp.items() if k!='note'})
PY
}
run base HD_X=0
run ag1 HD_MAC_AG=1
run ag1s2 HD_MAC_AG=1 HD_MAC_STAGES=2
run ag1s2A HD_MAC_AG=1 HD_MAC_STAGES=2 HD_PRIO=A
run ag1s2B HD_MAC_AG=1 HD_MAC_STAGES=2 HD_PRIO=0
