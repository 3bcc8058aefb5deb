import numpy as np, sys
a=np.load(sys.argv[1] if len(sys.argv)>1 else 'gpurun_out/timeline.npy')
def trim(x):
    out=[]
    for r in x:
        if r[3]==0: break
        out.append(r)
    return np.array(out)
def cut(x):
    for i in range(1,len(x)):
        if x[i,1] < x[i-1,1]-5: return x[:i]
    return x
mma=np.concatenate([cut(trim(a[0])), cut(trim(a[3]))]); mma=mma[np.argsort(mma[:,3])]; s0=trim(a[1]); s1=trim(a[2])
t0=mma[0,3]
def ev(x,e,t,j):
    m=(x[:,0]==e)&(x[:,1]==t)&(x[:,2]==j)
    return int(x[m][0,3]-t0) if m.any() else None
G=int(mma[:,2].max())+1
ts=sorted(set(mma[:,1]))[40:43]
for t in ts:
    base=ev(mma,1,t,G-1)
    print('t',t,'MMA:', ' '.join(f"j{j}[{ev(mma,1,t,j)-base}..{ev(mma,2,t,j)-base}]" for j in range(G-1,-1,-1)))
    for name,x,s in (('set0',s0,0),('set1',s1,1)):
        items=[]
        for j in range(G-1,-1,-1):
            if j%2!=s: continue
            f=ev(x,10+s,t,j); fr=ev(x,20+s,t,j); af=ev(x,30+s,t,j)
            items.append(f"j{j}: full{f-base if f else '-'} free{fr-base if fr else '-'} out{af-base if af else '-'}")
        ld=ev(x,40,t,0) if s==0 else None
        print('   ',name,' | '.join(items), ('load%d'%(ld-base)) if ld else '')
st=[ev(mma,1,t,G-1) for t in sorted(set(mma[:,1]))[40:60]]
st=[x for x in st if x is not None]
print('period', np.diff(st))
print('--- epilogue sub-events (relative to acc_full observe)')
for name,x,s in (('set0',s0,0),('set1',s1,1)):
    for t in ts[:2]:
        for j in range(G-1,-1,-1):
            if j%2!=s: continue
            f=ev(x,10+s,t,j)
            if f is None: continue
            row=[]
            for e,nm in ((50,'ld'),(20,'free'),(60,'math'),(70,'empty'),(80,'sts'),(30,'out')):
                v=ev(x,e+s,t,j)
                row.append(f"{nm}+{v-f}" if v is not None else f"{nm}-")
            print(name,'t',t,'j',j,' '.join(row))
