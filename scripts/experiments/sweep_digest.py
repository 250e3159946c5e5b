import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
sw=d['advance_sweep']
print(sys.argv[1], 'headline', round(d['roofline']['frac'],3), 'single', {k: round(v['single']['frac_hbm'],3) for k,v in sw.items() if k!='note'}, 'chained', {k: round(v['chained']['frac_hbm'],3) for k,v in sw.items() if k!='note'})
