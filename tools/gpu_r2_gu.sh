# gate/up + LM head on the cluster kernel with S=1 (VC_GEMM_CLUSTER_MIN=1) vs stream-K
for mn in 3 1; do for m in draft mixed; do
VC_GEMM_CLUSTER_MIN=$mn timeout 600 python tools/profile_step.py --mode $m --steps 8 --x 6 2>&1 | tail -1 | sed "s/^/min=$mn /"
done; done
VC_GEMM_CLUSTER_MIN=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_mixed_min1.csv python tools/profile_step.py --mode mixed --x 6 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launch_mixed_min1.csv')))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
st=[i for i,d in enumerate(data) if 'embed_norm' in d['Kernel Name']][-1]
for d in data[st:st+10]+data[-3:]:
    print(d['Kernel Name'].split('(')[0][-45:], d['Metric Value'], d['Grid Size'])
PY
