import sys, numpy as np
sys.path.insert(0, '.')
from tests import _golden as G
from oracle import cp_oracle as O
import paper_1205_2584_b200 as api
E = G.ensemble()
for key in ['e3_auto', 'e6_flm-a', 'e9_auto', 'e14_auto', 'e0_auto']:
    e = E[key]; variant = key.split('_', 1)[1]
    y = e['y']; r = int(e['rank'])
    print(key, y.shape, 'R', r, 'complex', np.iscomplexobj(y))
    res = api.fit(api.DenseTensor(y), api.FitConfig(rank=r, variant=variant, tol=1e-10, max_iters=40, seed=int(e['seed']), init='random'))
    ref = e['trace']
    got = np.array([[t.iter, t.relerr, t.mu, t.accepted] for t in res.trace])
    n = min(len(got), len(ref))
    print('  seq gpu', ''.join('A' if a else 'r' for a in got[:, 3]))
    print('  seq ref', ''.join('A' if a else 'r' for a in ref[:, 3]))
    print('  relerr diff', np.abs(got[:n, 1] - ref[:n, 1]).max(), ' first diffs', np.abs(got[:6, 1] - ref[:6, 1]))
    print('  mu ratio first', got[:6, 2] / ref[:6, 2])
    print('  relerr', ref[:4, 1], ref[-1, 1])
