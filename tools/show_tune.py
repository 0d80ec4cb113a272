import json, sys
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except Exception: print(l[:300]); continue
    if 'error' in d: print(d['env'], d['error'][-1500:]); continue
    print(d['env'])
    for k, v in d.items():
        if k == 'env': continue
        if isinstance(v, float): v = round(v, 2)
        elif isinstance(v, list): v = [round(x, 2) if isinstance(x, float) else x for x in v]
        elif isinstance(v, dict): v = {a: round(b, 2) for a, b in v.items()}
        print('   ', k, v)
