import sys
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, torch
import bench_workloads as bw
dev=torch.device('cuda',0)
model, tab, enc = bw.config3(dev)
rng = np.random.default_rng(77)
phrases,_=bw.gi.corpus('p5k_v1024')
tpf = bw.config3_targets(rng, tab.vocab_size, 200, phrases)
ts=[t for t in range(200) if tpf[t]>=0][:4]; bs=[t for t in range(200) if tpf[t]<0][:2]
for t in ts+bs:
    y=int(tpf[t]); e=enc[0,t:t+1]
    for ctx in (-1, 5, max(y,1)):
        lp=model.joint_logprobs(e, torch.tensor([[ctx]],device=dev))[0]
        top=torch.topk(lp,3)
        print(t,'y',y,'ctx',ctx,'lp[y]',round(float(lp[max(y,0)]),2),'lp[blank]',round(float(lp[0]),2),'top',[(int(i),round(float(v),2)) for v,i in zip(top.values,top.indices)])
