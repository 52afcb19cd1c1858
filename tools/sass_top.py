import csv,gzip,sys,collections
f=gzip.open(sys.argv[1],'rt'); next(f)
rd=csv.reader(f); hdr=next(rd)
ix={h:i for i,h in enumerate(hdr)}
rows=[r for r in rd if len(r)>10]
tot=sum(int(r[ix['# Samples']]) for r in rows)
texec=sum(int(r[ix['Instructions Executed']]) for r in rows)
print('total samples',tot,'inst executed',texec)
# stall totals
stalls=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
agg=collections.Counter()
for r in rows:
    for s in stalls: agg[s]+=int(r[ix[s]] or 0)
print(sorted(agg.items(), key=lambda kv:-kv[1])[:8])
# by opcode
byop=collections.Counter(); byop_n=collections.Counter()
for r in rows:
    op=r[ix['Source']].split()[0]
    if op.startswith('@'): op=r[ix['Source']].split()[1]
    op=op.split('.')[0]
    byop[op]+=int(r[ix['# Samples']]); byop_n[op]+=int(r[ix['Instructions Executed']])
print('by opcode (samples, executed):')
for k,v in byop.most_common(14): print('  ',k,v,round(100*v/tot,1),'%', byop_n[k], round(100*byop_n[k]/texec,1),'%')
n=int(sys.argv[2]) if len(sys.argv)>2 else 25
print('top instructions:')
for i,r in sorted(enumerate(rows), key=lambda ir:-int(ir[1][ix['# Samples']]))[:n]:
    top=sorted(((int(r[ix[s]] or 0),s) for s in stalls), reverse=True)[:2]
    print(i, r[ix['Source']].strip()[:60], r[ix['# Samples']], r[ix['Instructions Executed']], top)
