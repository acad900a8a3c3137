import sys, numpy as np, time
sys.path.insert(0, '/root/repo')
from oracle import cp_oracle as O
from tests import _golden as G
from paper_1205_2584_b200 import synth
mode = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else 'fit_c1_s0_auto'
d = G.load_fit(name)
y = synth.make_tensor(G.synth_config(d), 0)
cfg = O.OracleConfig(rank=d['rank'], tau=d['tau'], tol=0.0, max_iters=d['max_iters'], seed=0)
if mode == 'solve':
    class LUB:
        def __init__(self, phi, k=None): self.lu = __import__('scipy').linalg.lu_factor(phi); self.k = k
        def __matmul__(self, w):
            z = __import__('scipy').linalg.lu_solve(self.lu, w)
            return z if self.k is None else self.k @ z
    def b_core(g, mu, use_kinv):
        psi = __import__('scipy').linalg.block_diag(*O.psi_diag_blocks(g, mu))
        if use_kinv: return LUB(O.kernel_inverse(g) + psi)
        k = O.kernel_matrix(g); return LUB(np.eye(k.shape[0]) + psi @ k, k)
    O.b_core = b_core
elif mode == 'perturb':
    orig = O.relative_error
    def rel(y, f):
        v = orig(y, f); return v * (1 + 1e-14)
    O.relative_error = rel
t = time.time()
res = O.fit_lm(y, cfg)
v = O.stack(res.factors)
print(name, mode, 'seq equal', res.accepted == G.accept_seq(d['trace']), 'final relerr diff', res.final_relerr - d['trace'][-1,1],
      'factor rel diff', np.linalg.norm(v - d['factors'])/np.linalg.norm(d['factors']), 'time', time.time()-t)
tr = np.array([e for (_, e, _, _) in res.trace])
print('relerr diffs by iter', np.abs(tr - d['trace'][:,1])[::5])
