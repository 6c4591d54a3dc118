"""Timeline of one attention CTA from an -DIG_ATTN_TRACE build (clock64 per event)."""
import sys
for f in sys.argv[1:]:
    rows=[l.split() for l in open(f) if l.startswith("TR")]
    ev={}
    for r in rows:
        t,j=int(r[1]),int(r[2]); ev[(t,j)]=[int(x) for x in r[3:]]
    base=min(min(x for x in e if x>0) for e in ev.values())
    print(f)
    n = len(ev[(0,0)])
    # merged event list for j in 10..12
    evs=[]
    names={0:"MMA: wait P",1:"MMA: P full",2:"SM: wait S",3:"SM: S seen",4:"SM: done",5:"SM: exp start",6:"SM: exp end",7:"MMA: V landed",8:"MMA: S(j+1) issued",9:"MMA: wait V"}
    for j in range(10,13):
        for t in range(2):
            for k in range(n):
                x=ev[(t,j)][k]
                if x>0 and not (k in (7,9) and t==1): evs.append((x-base,t,j,names.get(k, str(k))))
    evs.sort()
    for x,t,j,nm in evs: print(f"{x:7d}  t{t} j{j:2d}  {nm}")
    for t in range(2):
        ps=[ev[(t,j+1)][3]-ev[(t,j)][3] for j in range(5,30)]
        print("period t",t, sum(ps)/len(ps))
