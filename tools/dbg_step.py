import sys, numpy as np
sys.path.insert(0, '.')
from tests import _golden as G
from oracle import cp_oracle as O
import paper_1205_2584_b200 as api
np.set_printoptions(precision=4, linewidth=150)
for cname in ['case0', 'case6']:
    c = G.unit_cases()[cname]; dims = tuple(int(x) for x in c['dims']); r = int(c['rank'])
    fac = G.split_stacked(c['factors'], dims, r); y = np.asfortranarray(c['y'])
    g = O.gram_cache(fac); M = [O.mttkrp(y, fac, n) for n in range(1, len(dims)+1)]
    mu = 0.1
    damped = [O.damped_factor(M[n], g, n, mu) for n in range(len(dims))]
    w = O.projected_residual(fac, g, damped, mu)
    b = O.core_matrix(g, mu, 'flm-b')
    F = O.frontal_slices(b @ w, len(dims), r)
    cand0 = O.factored_update(fac, damped, F, g, mu)
    gpu = api.flm_step(api.DenseTensor(y), api.KruskalModel(fac), mu, 'flm-b', refine_steps=0)
    for n in range(len(dims)):
        print(cname, 'mode', n, 'max |gpu-oracle|', np.abs(gpu.factors[n]-cand0[n]).max())
        # recover E_gpu = pinv(A)(cand - D)
        E = np.linalg.lstsq(fac[n], gpu.factors[n]-damped[n], rcond=None)[0]
        Eo = np.eye(r) - (F[n] + g.excl[n].T) @ np.linalg.inv(g.excl[n].T + mu*np.eye(r))
        print('  E gpu\n', E, '\n  E oracle\n', Eo)
        Fg = (np.eye(r) - E) @ (g.excl[n].T + mu*np.eye(r)) - g.excl[n].T
        print('  F gpu\n', Fg, '\n  F oracle\n', F[n])
    print('w', w)
