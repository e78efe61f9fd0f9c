import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; data=rows[2:]
ix={k:i for i,k in enumerate(h)}
S=ix['Source']; IE=ix['Instructions Executed']
mix={}
for r in data:
    if not r[S]: continue
    toks=r[S].split()
    op=toks[0]
    if op.startswith('@'): op=toks[1] if len(toks)>1 else op
    op=op.split('.')[0]
    mix[op]=mix.get(op,0)+int(r[IE] or 0)
tot=sum(mix.values())
half={'DADD','DFMA','DMUL','FFMA2','FADD2','FMUL2','DSETP'}
hw=sum(v for k,v in mix.items() if k in half)
print('total',tot,'half-rate',hw,'weighted cycles',tot+hw)
for k,v in sorted(mix.items(),key=lambda x:-x[1])[:14]: print(f'  {k:10s} {v:12d} {100*v/tot:5.1f}%')
