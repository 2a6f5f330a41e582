import json,sys
for f in sys.argv[1:]:
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, 'ERR', e); continue
    r=d.get('roofline',{})
    print(f, 'value=%.3f'%d['value'], 'ms=%.2f'%d.get('ms_per_step',0), 'e2e=%s'%(d.get('e2e',{}).get('value')), 'rel=%s'%d.get('rel_err'), d.get('selected_blocks'))
    if r: print('   roof %s %.1f/%.1f %s frac=%.3f'%(r.get('kernel'),r.get('achieved',0),r.get('peak',0),r.get('unit'),r.get('frac',0)), d.get('clocks'))
    k=d.get('kernels_per_step',{})
    for n,v in sorted(k.items(), key=lambda x:-x[1]['ms'])[:16]: print('   %-28s %8.3f ms x%d'%(n,v['ms'],v['scopes']), ('%.0f GB/s'%(v['bytes']/v['ms']/1e6) if v['bytes'] else ''), ('%.0f TF/s'%(v['flops']/v['ms']/1e9) if v['flops'] else ''))
