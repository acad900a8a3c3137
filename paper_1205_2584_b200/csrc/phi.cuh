// The NR^2 x NR^2 core system of the fLM step (hessian.py:62-119, 185-211; solver.py:143-169).
//
//   flm-b (K invertible):  Phi_2 = K~ + Psi,      B w = Phi_2^{-1} w
//   flm-a (always):        Phi_1 = I + Psi K,     B w = K Phi_1^{-1} w
// with Psi = blkdiag((Gamma_n + mu I)^{-1} kron C_n)  (NOT transposed, hessian.py:191),
//      K_{nm}  = (1-delta) P_R diag(vec Gamma^(n,m))            (hessian.py:62-68)
//      K~_{nm} = (1/(N-1) - delta) diag(vec(C_n o C_m / Gamma)) P_R   (hessian.py:108-119)
// Phi_2 is Hermitian indefinite and Phi_1 non-symmetric, so the solve is an LU with partial
// pivoting (lu.cuh), exactly the family the reference's np.linalg.inv / solve uses.  Instead of
// forming B = Phi^{-1} explicitly (hessian.py:207) the factors are kept and B w is applied by
// triangular solves (3 right-hand sides per iteration: main step + 2 refinements).
#pragma once
#include "cpf_common.cuh"

namespace cpf {

// Assemble Phi (column-major, ld = nB) for the variant in st->use_kinv.  One thread per entry.
template <class T>
__global__ void k_phi_assemble(T* __restrict__ Phi, int N, int R, const T* __restrict__ Cg,
                               const T* __restrict__ Gi, const T* __restrict__ pair, const T* __restrict__ full,
                               const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (gate_running && st->stopped) return;
  if (st->err_code) return;
  if (gate_running == 2 && st->rej_grow) return;  // after a rho <= 0 rejection the speculated system is used
  if (lu_gated(st, gate_running == 3 ? 3 : 0)) return;
  const int R2 = R * R;
  const int64_t nB = (int64_t)N * R2;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nB * nB) return;
  const int64_t p = idx % nB, q = idx / nB;
  const int n = (int)(p / R2), m = (int)(q / R2);
  const int pl = (int)(p % R2), ql = (int)(q % R2);
  const int a1 = pl % R, b1 = pl / R;  // row (a' + R b')
  const int c1 = ql % R, d1 = ql / R;  // col (c' + R d')
  T v;
  if (st->use_kinv) {
    T k = zero_of<T>();
    // K~ nonzero iff ql == b1 + R*a1 (row pl = a + R b, col b + R a)
    if (ql == b1 + R * a1) {
      const double coeff = 1.0 / (N - 1) - (n == m ? 1.0 : 0.0);
      const int e = a1 + R * b1;
      T d = dvd(mul(Cg[(int64_t)n * R2 + e], Cg[(int64_t)m * R2 + e]), full[e]);
      k = scale(d, coeff);
    }
    if (n == m) {
      T psi = mul(Gi[(int64_t)n * R2 + b1 + R * d1], Cg[(int64_t)n * R2 + a1 + R * c1]);
      v = add(k, psi);
    } else {
      v = k;
    }
  } else {
    // I + Psi K ; (Psi_n K_nm)[pl, ql = b + R a] = Psi_n[pl, a + R b] * Gamma^(n,m)[b, a]
    T pk = zero_of<T>();
    if (n != m) {
      const int b = ql % R, a = ql / R;
      // Psi_n[a1 + R b1, a + R b] = Gi_n[b1, b] * C_n[a1, a]
      T psi = mul(Gi[(int64_t)n * R2 + b1 + R * b], Cg[(int64_t)n * R2 + a1 + R * a]);
      pk = mul(psi, pair[((int64_t)n * N + m) * R2 + b + R * a]);
    }
    v = add(from_real<T>(p == q ? 1.0 : 0.0), pk);
  }
  Phi[idx] = v;
}

// Fault injection (test hook CPF_TEST_SINGULAR=t): zero column 0 of the core system factored for
// iteration t (offset: 1 for the next step's system, 2 for the speculated rejection branch's) so its
// LU meets an exactly zero pivot -- the reference's LinAlgError("Singular matrix") stop.
template <class T>
__global__ void k_test_zero_col(T* __restrict__ Phi, int nB, const LmDeviceState* st, int offset) {
  pdl_wait();
  if (st->test_singular_iter == 0 || st->iter + offset != st->test_singular_iter) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nB; i += gridDim.x * blockDim.x) Phi[i] = zero_of<T>();
}

// flm-a: f = K z  ((K z)_n[a + R b] = sum_{m != n} Gamma^(n,m)[b, a] z_m[b + R a]); flm-b: f = z.
template <class T>
__global__ void k_apply_k(const T* __restrict__ z, int N, int R, const T* __restrict__ pair, T* __restrict__ f,
                          const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (gate_running && st->stopped) return;
  if (st->err_code) return;
  const int R2 = R * R;
  const int64_t nB = (int64_t)N * R2;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nB) return;
  if (st->use_kinv) { f[p] = z[p]; return; }
  const int n = (int)(p / R2), pl = (int)(p % R2);
  const int a = pl % R, b = pl / R;
  T acc = zero_of<T>();
  bool first = true;
  for (int m = 0; m < N; ++m) {
    if (m == n) continue;
    T v = mul(pair[((int64_t)n * N + m) * R2 + b + R * a], z[(int64_t)m * R2 + b + R * a]);
    acc = first ? v : add(acc, v);
    first = false;
  }
  f[p] = acc;
}

}  // namespace cpf
