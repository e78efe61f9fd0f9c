import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; data=rows[2:]
ix={k:i for i,k in enumerate(h)}
A=ix['Address']; S=ix['Source']; NS=ix['# Samples']; IE=ix['Instructions Executed']
tot=sum(int(r[NS] or 0) for r in data); totI=sum(int(r[IE] or 0) for r in data)
print('total samples',tot,'total inst',totI)
# segment into regions by branches targets: print cumulative by blocks of backward BRA
seg=[];cur=[]
for r in data:
    cur.append(r)
    op=r[S].split()[0] if r[S] else ''
    if 'BRA' in r[S] or 'EXIT' in r[S] or 'RET' in r[S] or 'BAR' in r[S] or 'SYNCS' in r[S] or 'WARPSYNC' in r[S]:
        seg.append(cur);cur=[]
if cur: seg.append(cur)
stalls=[k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
for s in seg:
    n=sum(int(r[NS] or 0) for r in s); ie=sum(int(r[IE] or 0) for r in s)
    if n<tot*0.004: continue
    ops={}
    for r in s:
        op=r[S].split()[0].split('.')[0] if r[S] else ''
        ops[op]=ops.get(op,0)+1
    top=sorted(ops.items(),key=lambda x:-x[1])[:5]
    st={k:sum(int(r[ix[k]] or 0) for r in s) for k in stalls}
    stt=sorted(st.items(),key=lambda x:-x[1])[:4]
    print(f"{s[0][A]}..{s[-1][A]} n_instr {len(s):5d} samples {n:7d} ({100*n/tot:5.1f}%) exec {ie:10d} ({100*ie/totI:5.1f}%) ops {top} stalls {stt}")
