import torch, json, sys
sys.path.insert(0, '.')
import paper_2403_01876_b200 as dv
L,H,D,B,P,S=40,40,128,8,1000,2048
k6=torch.empty((L,B,H,D//8,S,8),dtype=torch.int16,device='cuda'); v=torch.empty((L,B,H,S,D),dtype=torch.int16,device='cuda')
k5=torch.empty((L,B,H,S,D),dtype=torch.int16,device='cuda')
c6=dv.cache(k6,v); c5=dv.cache(k5,v)
ctx=dv.dv_create(0)
dbuf=torch.empty(2*B*H*P*D,dtype=torch.int16,device='cuda'); ep=dv.endpoint_of(dbuf)
st=torch.cuda.current_stream()
def t(fn,n=50,reps=7):
    return sorted(t1(fn,n) for _ in range(reps))[reps//2]
def t1(fn,n):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n): fn()
    b.record(st); torch.cuda.synchronize(); return a.elapsed_time(b)/n*1e3
nb=2*B*H*P*D*2
for name,c in (("ft6d",c6),("kv5d",c5)):
    us=t(lambda: dv.dv_scatter(ctx,c,dv.region(3,4,0,B,0,P),ep,0))
    print(name, "prompt pack us", us, "frac", 2*nb/us/1e3/6534.8)
# K only vs V only timing via head-subsets isn't separable; time region of half heads
