import json, sys
for path in sys.argv[1:]:
    print("==", path)
    for l in open(path):
        if not l.startswith('{'):
            print(l.strip()); continue
        d = json.loads(l)
        per = d['solve_ms'] / max(d['inner_iters_total'], 1) * 1e3 if d['inner_iters_total'] else 0
        print(f"{d['method']:4s} rep{d['rep']} st={d['status']} outer={d['outer_iters']} inner={d['inner_iters_total']} "
              f"setup={d['setup_ms']:.3f} solve={d['solve_ms']:.3f}ms us/step={per:.3f} err={d.get('err')} hot={[round(x,3) for x in d['hot_ms']]}")
