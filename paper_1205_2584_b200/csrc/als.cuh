// ALS / ALS with line search on the engine: the R x R pseudo-inverse of a
// Hermitian PSD Gram product and the per-mode factor update.  The tensor reads (one MTTKRP per mode
// per sweep) reuse the fLM engine's pass A / pass B; these kernels are the R x R tail.
//
//   pinv_psd(G)  = V diag(1/w, w > eps*R*max(w, 0)) V^H     cpfast/kruskal.py:245-254
//   als_step     A_n <- M_n pinv_psd(Gamma^(n))^T, n = 1..N   cpfast/kruskal.py:257-265
//   line search  cand = A_prev + s (A_als - A_prev)           cpfast/kruskal.py:268-293
#pragma once

#include "cpf_common.cuh"

// Largest R the single-CTA eigen-solver takes (2 m x m tiles of T in shared memory, m = R rounded
// to even): 64 -> 128 KB complex, 64 KB real.
constexpr int kPinvMaxR = 64;

template <class T>
__host__ __device__ constexpr size_t pinv_smem_bytes(int R) {
  return (size_t)2 * (R + (R & 1)) * (R + (R & 1)) * sizeof(T) + (size_t)(R + 2) * (2 * sizeof(double) + sizeof(T) + 2 * sizeof(int));
}

// Eigen-decomposition of the Hermitian R x R matrix G (column-major; the lower triangle is read, as
// LAPACK ?syevd/?heevd with UPLO='L' under np.linalg.eigh) by cyclic two-sided Jacobi with the
// round-robin (circle) ordering: each round rotates m/2 disjoint (p, q) pairs in parallel --
// A <- U^H A U with U block-diagonal over the pairs, V <- V U.  The 2 x 2 Hermitian block
// [[a, b], [b*, d]], b = |b| e^{i phi}, is diagonalised by U = diag(1, e^{-i phi}) [[c, s], [-s, c]]
// (Golub & Van Loan sym.schur2 on the phase-normalised real block).  A pair is rotated while
// |a_pq| > eps sqrt(|a_pp a_qq|) (the relative-accuracy criterion of one-sided Jacobi); the sweep
// loop ends at the first sweep with no rotation.  Then the pseudo-inverse with kruskal.py's
// truncation.  One CTA: the matrices are at most 64 x 64.
template <class T>
__global__ void __launch_bounds__(256) k_pinv_psd(const T* __restrict__ G, int R, T* __restrict__ out) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = R + (R & 1);  // odd R: index R is a zero dummy, never rotated (a_pq = 0)
  const int np = m / 2;
  T* a = reinterpret_cast<T*>(smem_raw);
  T* v = a + m * m;
  double* rc = reinterpret_cast<double*>(v + m * m);
  double* rs = rc + np + 1;
  T* rph = reinterpret_cast<T*>(rs + np + 1);
  int* rp = reinterpret_cast<int*>(rph + np + 1);
  int* rq = rp + np + 1;
  __shared__ int rotated;
  __shared__ double s_wmax;
  __shared__ double inv_w[kPinvMaxR];
  const int tid = threadIdx.x, nthr = blockDim.x;
  constexpr double eps = 2.220446049250313e-16;
  for (int e = tid; e < m * m; e += nthr) {
    const int i = e % m, j = e / m;
    T x = zero_of<T>();
    if (i < R && j < R) x = (i >= j) ? G[i + (int64_t)R * j] : cj(G[j + (int64_t)R * i]);
    if (i == j) x = from_real<T>(re(x));
    a[e] = x;
    v[e] = from_real<T>(i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  if (m >= 2) {
    for (int sweep = 0; sweep < 64; ++sweep) {
      if (tid == 0) rotated = 0;
      __syncthreads();
      for (int r = 0; r < m - 1; ++r) {
        for (int k = tid; k < np; k += nthr) {
          int p, q;
          if (k == 0) {
            p = r; q = m - 1;
          } else {
            p = (r + k) % (m - 1);
            q = (r - k + m - 1) % (m - 1);
          }
          if (p > q) { const int t = p; p = q; q = t; }
          const T apq = a[p + m * q];
          const double app = re(a[p + m * p]), aqq = re(a[q + m * q]);
          const double mag = modulus(apq);
          double c = 1.0, sn = 0.0;
          T ph = from_real<T>(1.0);
          if (mag > 1e-300 && mag > eps * sqrt(fabs(app * aqq))) {
            ph = scale(apq, 1.0 / mag);
            const double tau = (aqq - app) / (2.0 * mag);
            double t;
            if (fabs(tau) > 1e150) t = 0.5 / tau;
            else t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            sn = t * c;
            rotated = 1;
          }
          rc[k] = c; rs[k] = sn; rph[k] = ph; rp[k] = p; rq[k] = q;
        }
        __syncthreads();
        // columns: A <- A U, V <- V U;  U = [[c, s], [-s conj(ph), c conj(ph)]] on (p, q)
        for (int e = tid; e < np * m; e += nthr) {
          const int k = e / m, i = e % m;
          const double sn = rs[k];
          if (sn == 0.0) continue;
          const double c = rc[k];
          const int p = rp[k], q = rq[k];
          const T phc = cj(rph[k]);
          {
            const T ap = a[i + m * p], aq = mul(phc, a[i + m * q]);
            a[i + m * p] = sub(scale(ap, c), scale(aq, sn));
            a[i + m * q] = add(scale(ap, sn), scale(aq, c));
          }
          {
            const T vp = v[i + m * p], vq = mul(phc, v[i + m * q]);
            v[i + m * p] = sub(scale(vp, c), scale(vq, sn));
            v[i + m * q] = add(scale(vp, sn), scale(vq, c));
          }
        }
        __syncthreads();
        // rows: A <- U^H A;  U^H = [[c, -s ph], [s, c ph]]; the rotated entry is set to zero
        for (int e = tid; e < np * m; e += nthr) {
          const int k = e / m, j = e % m;
          const double sn = rs[k];
          if (sn == 0.0) continue;
          const double c = rc[k];
          const int p = rp[k], q = rq[k];
          const T ph = rph[k];
          const T ap = a[p + m * j], aq = mul(ph, a[q + m * j]);
          T np_ = sub(scale(ap, c), scale(aq, sn));
          T nq_ = add(scale(ap, sn), scale(aq, c));
          if (j == q) np_ = zero_of<T>();
          if (j == p) nq_ = zero_of<T>();
          if (j == p) np_ = from_real<T>(re(np_));
          if (j == q) nq_ = from_real<T>(re(nq_));
          a[p + m * j] = np_;
          a[q + m * j] = nq_;
        }
        __syncthreads();
      }
      const int any = rotated;
      __syncthreads();
      if (!any) break;
    }
  }
  // pseudo-inverse: eigenvalues w_p = a_pp (p < R), cutoff eps * R * max(max w, 0)
  if (tid == 0) {
    double w = -INFINITY;
    for (int p = 0; p < R; ++p) w = fmax(w, re(a[p + m * p]));
    s_wmax = w;
  }
  __syncthreads();
  const double cutoff = eps * R * fmax(s_wmax, 0.0);
  for (int p = tid; p < R; p += nthr) {
    const double w = re(a[p + m * p]);
    inv_w[p] = w > cutoff ? 1.0 / w : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < R * R; e += nthr) {
    const int i = e % R, j = e / R;
    T acc = zero_of<T>();
    for (int p = 0; p < R; ++p) {
      if (inv_w[p] == 0.0) continue;
      fma_acc(acc, scale(v[i + m * p], inv_w[p]), cj(v[j + m * p]));
    }
    out[e] = acc;
  }
}

// out (I x R, column-major) = Mn Pinv^T  (kruskal.py:264: m @ pinv_psd(gamma).T, no conjugation)
template <class T>
__global__ void k_als_factor(const T* __restrict__ Mn, const T* __restrict__ P, int64_t I, int R, T* __restrict__ out) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sp = reinterpret_cast<T*>(smem_raw);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) sp[e] = P[e];
  __syncthreads();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= I * R) return;
  const int64_t i = idx % I;
  const int c = (int)(idx / I);
  T acc = mul(Mn[i], sp[c]);  // Pinv^T[k, c] = Pinv[c, k] = sp[c + R k]
  for (int k = 1; k < R; ++k) fma_acc(acc, Mn[i + I * k], sp[c + R * k]);
  out[idx] = acc;
}

// line-search candidate (kruskal.py:283-287): out = hp + s * (ha - hp), rounded step by step
template <class T>
__global__ void k_als_extrap(const T* __restrict__ hp, const T* __restrict__ ha, double s, int64_t n, T* __restrict__ out) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T p = hp[i], q = ha[i];
  if constexpr (ScalarTraits<T>::kComplex) {
    const double dx = __dsub_rn(q.x, p.x), dy = __dsub_rn(q.y, p.y);
    out[i] = T{__dadd_rn(p.x, __dmul_rn(s, dx)), __dadd_rn(p.y, __dmul_rn(s, dy))};
  } else {
    out[i] = __dadd_rn(p, __dmul_rn(s, __dsub_rn(q, p)));
  }
}
