// Factor-sized (T x R) and core-sized (R x R) kernels of one fLM iteration.
//
// Stacked layout: every per-mode I_n x R matrix (factors, MTTKRPs, damped factors, gradient,
// refinement vectors) lives column-major at offset R*sum_{k<n} I_k of one buffer, which is
// exactly the reference's stacked vector convention (kruskal.py:70-82).  R x R matrices are
// column-major, one per mode.
//
// All reductions are fixed-order (deterministic); every kernel reads the LM state from device
// memory so one iteration is a fixed launch sequence.
#pragma once
#include "cpf_common.cuh"

namespace cpf {

constexpr int kMaxModes = 8;

struct Modes {
  int N;
  int R;
  int64_t dims[kMaxModes];
  int64_t offs[kMaxModes];  // element offsets in the stacked buffer
};

// Kernel gating.  kAlways: unconditional (preamble); kRunning: skip once the fit stopped;
// kOnAccept: only while an accepted candidate is being committed (flags->pending_accept);
// kOnDirect / kOnCurDirect: the guard-band direct residual of the candidate / current model.
// kOnRejectPrev: the previous decision was a rho <= 0 rejection (its core system was speculated);
// kOnCoreNeeded: running and not kOnRejectPrev (the fork must factor the next core system).
enum Gate : int { kAlways = 0, kRunning = 1, kOnAccept = 2, kOnDirect = 3, kOnCurDirect = 4, kOnRejectPrev = 5,
                  kOnCoreNeeded = 6 };

// Ozaki accuracy guard (tensor_pass_oz.cuh): per pass (0 = A, 1 = B) and operand column r,
// oz_bad[pass][r] != 0 when that column of this launch's K x R operand is outside the int8 split's
// accuracy envelope; the pass then runs in fp64 instead.  Composite gates: kGateIfOzOk / kGateIfOzBad
// OR-ed into a base gate (bit kGateOzPass selects the pass) additionally require every / some column
// flag clear / set.
constexpr int kOzGuardCols = 32;
struct DevFlags {
  int pending_accept;
  int need_direct;
  int need_cur_direct;
  int oz_fallbacks;                   // passes this fit that ran in fp64 because of the guard
  int oz_bad[2][kOzGuardCols];
};
constexpr int kGateBaseMask = 0xff;
constexpr int kGateIfOzOk = 0x100;
constexpr int kGateIfOzBad = 0x200;
constexpr int kGateOzPass = 0x400;  // set: pass B's flags

__device__ __forceinline__ bool gate_open(const LmDeviceState* st, const DevFlags* fl, int gate) {
  if (gate & (kGateIfOzOk | kGateIfOzBad)) {
    const int* f = fl->oz_bad[(gate & kGateOzPass) ? 1 : 0];
    int any = 0;
#pragma unroll 4
    for (int r = 0; r < kOzGuardCols; ++r) any |= f[r];
    if ((gate & kGateIfOzOk) ? any != 0 : any == 0) return false;
    gate &= kGateBaseMask;
  }
  if (gate == kAlways) return true;
  if (gate == kRunning) return st->stopped == 0;
  if (gate == kOnAccept) return fl->pending_accept != 0;
  if (gate == kOnDirect) return fl->need_direct != 0;
  if (gate == kOnRejectPrev) return st->stopped == 0 && st->err_code == 0 && st->iter > 0 && st->rej_grow;
  if (gate == kOnCoreNeeded) return st->stopped == 0 && !st->rej_grow;
  return fl->need_cur_direct != 0;
}

// ------------------------------------------------------------------------------------------
// Cross Grams: out[n][r + R s] = sum_i conj(X_n[i, r]) * Y_n[i, s]   (kruskal.py:110, solver.py:136,
// hessian.py:314,340).  grid (R*R, N); deterministic block tree.
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_cross_gram(const T* __restrict__ X, const T* __restrict__ Yv, Modes md, T* __restrict__ out,
                             const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  __shared__ T scratch[32];
  const int n = blockIdx.y;
  const int R = md.R;
  const int rs = blockIdx.x;
  const int r = rs % R, s = rs / R;
  const int64_t I = md.dims[n];
  const T* xr = X + md.offs[n] + I * r;
  const T* ys = Yv + md.offs[n] + I * s;
  T acc = zero_of<T>();
  for (int64_t i = threadIdx.x; i < I; i += blockDim.x) fma_cacc(acc, xr[i], ys[i]);
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) out[(int64_t)n * R * R + r + (int64_t)R * s] = acc;
}

// Hadamard products (kruskal.py:112-123): excl[n] = prod_{k!=n} C_k, pair[n][m] = prod_{k!=n,m} C_k
// (pair[n][n] = excl[n], ones if empty), full = prod_k C_k.  Products in ascending k like reduce().
template <class T>
__global__ void k_hadamards(const T* __restrict__ Cg, int N, int R, T* __restrict__ excl, T* __restrict__ pair,
                            T* __restrict__ full, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int R2 = R * R;
  if (e >= R2) return;
  auto prod_skip = [&](int s1, int s2) {
    T v = from_real<T>(1.0);
    bool first = true;
    for (int k = 0; k < N; ++k) {
      if (k == s1 || k == s2) continue;
      T c = Cg[(int64_t)k * R2 + e];
      v = first ? c : mul(v, c);
      first = false;
    }
    return v;
  };
  for (int n = 0; n < N; ++n) {
    T ex = prod_skip(n, n);
    excl[(int64_t)n * R2 + e] = ex;
    for (int m = 0; m < N; ++m) pair[((int64_t)n * N + m) * R2 + e] = (m == n) ? ex : prod_skip(n, m);
  }
  full[e] = prod_skip(-1, -1);
}

// kernel_is_invertible (hessian.py:81-94): every |Gamma^(n,m)| (n != m) > 1e-10 * max.
// Single block.  Writes st->use_kinv for the variant in use; the flm-b-with-singular-K error is
// raised by the next step (solver.py:146-147).
template <class T>
__global__ void k_kernel_flag(const T* __restrict__ pair, int N, int R, LmDeviceState* st, const DevFlags* fl,
                              int gate, int* kinv_ok_out) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  __shared__ double smax[32], smin[32];
  const int R2 = R * R;
  double vmax = 0.0, vmin = INFINITY;
  for (int n = 0; n < N; ++n)
    for (int m = 0; m < N; ++m) {
      if (n == m) continue;
      for (int e = threadIdx.x; e < R2; e += blockDim.x) {
        double a = modulus(pair[((int64_t)n * N + m) * R2 + e]);
        vmax = fmax(vmax, a);
        vmin = fmin(vmin, a);
      }
    }
  for (int o = 16; o > 0; o >>= 1) {
    vmax = fmax(vmax, __shfl_down_sync(0xffffffffu, vmax, o));
    vmin = fmin(vmin, __shfl_down_sync(0xffffffffu, vmin, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) { smax[wid] = vmax; smin[wid] = vmin; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double top = 0.0, low = INFINITY;
    for (int w = 0; w < nw; ++w) { top = fmax(top, smax[w]); low = fmin(low, smin[w]); }
    int ok = (N >= 2) && (top != 0.0) && (low > 1e-10 * top);
    *kinv_ok_out = ok;
    // variant: 0 auto, 1 flm-a, 2 flm-b
    st->use_kinv = (st->variant == 1) ? 0 : (st->variant == 2 ? 1 : ok);
  }
}

// ------------------------------------------------------------------------------------------
// Damped Gamma inverses: Gti[n] = (Gamma_n^T + mu I)^{-1} (solver.py:119,134,181; hessian.py:336)
// and Gi[n] = (Gamma_n + mu I)^{-1} (hessian.py:191).  Gauss-Jordan with partial pivoting, one
// block per (mode, which).  A zero pivot flags numpy's LinAlgError("Singular matrix").
// Also raises the deferred flm-b/singular-K error for this iteration.
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_damped_inverses(const T* __restrict__ excl, int N, int R, T* __restrict__ Gti, T* __restrict__ Gi,
                                  LmDeviceState* st, const DevFlags* fl, int gate, const int* kinv_ok,
                                  const double* mu_override, int* sing_out = nullptr) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* a = reinterpret_cast<T*>(smem_raw);  // R x 2R augmented, column-major (ld = R)
  __shared__ int piv_s;
  __shared__ int sing_s;
  const int n = blockIdx.x % N;
  const int transposed = blockIdx.x / N == 0;  // first N blocks: Gti (transposed)
  const double mu = mu_override ? *mu_override : st->mu;
  const int R2 = R * R;
  const T* g = excl + (int64_t)n * R2;
  for (int e = threadIdx.x; e < 2 * R2; e += blockDim.x) {
    int i = e % R, j = e / R;
    T v;
    if (j < R) {
      v = transposed ? g[j + R * i] : g[i + R * j];
      if (i == j) v = add(v, from_real<T>(mu));
    } else {
      v = from_real<T>((i == j - R) ? 1.0 : 0.0);
    }
    a[i + R * j] = v;
  }
  if (threadIdx.x == 0) sing_s = 0;
  __syncthreads();
  for (int k = 0; k < R; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      double best = pivmag(a[k + R * k]);
      for (int i = k + 1; i < R; ++i) {
        double v = pivmag(a[i + R * k]);
        if (v > best) { best = v; p = i; }
      }
      piv_s = p;
      if (best == 0.0) sing_s = 1;
    }
    __syncthreads();
    if (sing_s) break;
    const int p = piv_s;
    if (p != k)
      for (int j = threadIdx.x; j < 2 * R; j += blockDim.x) {
        T t = a[k + R * j];
        a[k + R * j] = a[p + R * j];
        a[p + R * j] = t;
      }
    __syncthreads();
    const T pv = a[k + R * k];
    for (int j = threadIdx.x; j < 2 * R; j += blockDim.x) a[k + R * j] = dvd(a[k + R * j], pv);
    __syncthreads();
    for (int e = threadIdx.x; e < R * 2 * R; e += blockDim.x) {
      int i = e % R, j = e / R;
      if (i == k || j == k) continue;
      T f = a[i + R * k];
      fms_acc(a[i + R * j], f, a[k + R * j]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < R; i += blockDim.x)
      if (i != k) a[i + R * k] = zero_of<T>();
    __syncthreads();
  }
  T* out = (transposed ? Gti : Gi) + (int64_t)n * R2;
  for (int e = threadIdx.x; e < R2; e += blockDim.x) out[e] = a[e + R2];
  if (threadIdx.x == 0) {
    if (sing_s && sing_out) *sing_out = 1;  // speculative branch: reported if it is taken
    else if (sing_s && st->err_code == 0) { st->err_code = kErrSingular; }
    if (blockIdx.x == 0 && kinv_ok && st->variant == 2 && !*kinv_ok && st->err_code == 0)
      st->err_code = kErrKernelSingular;
  }
}

// ------------------------------------------------------------------------------------------
// Tall-skinny linear combination, per mode n (rows of the stacked buffer):
//   out_n = X1_n op(S1_n) + coef3 * X3_n + X2_n op(S2_n) [+ X4_n]
// op(S) = S, or S^T when the transpose bit is set.  Any of X1/X2/X3/X4 may be null.  S matrices
// are R x R column-major per mode (stride sstride; 0 = one matrix for all modes).
// coef3 < 0 selects the damping mu from the state (the mu*x term of hessian.py:317).
// ------------------------------------------------------------------------------------------
struct TallArgs {
  const void* X1; const void* S1; int t1; int64_t s1stride;
  const void* X2; const void* S2; int t2; int64_t s2stride;
  const void* X3; double coef3; int coef3_mu;
  const void* X4; double coef4;
  int neg1;
  void* out;
};

template <class T>
__global__ void k_tall(TallArgs a, Modes md, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = md.R;
  const int R2 = R * R;
  T* s1 = reinterpret_cast<T*>(smem_raw);
  T* s2 = s1 + R2;
  const int n = blockIdx.y;
  const T* S1 = a.S1 ? static_cast<const T*>(a.S1) + a.s1stride * n : nullptr;
  const T* S2 = a.S2 ? static_cast<const T*>(a.S2) + a.s2stride * n : nullptr;
  for (int e = threadIdx.x; e < R2; e += blockDim.x) {
    int i = e % R, j = e / R;
    if (S1) s1[e] = a.t1 ? S1[j + R * i] : S1[e];
    if (S2) s2[e] = a.t2 ? S2[j + R * i] : S2[e];
  }
  __syncthreads();
  const int64_t I = md.dims[n];
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= I * R) return;
  const int64_t i = idx % I;
  const int c = (int)(idx / I);
  const int64_t base = md.offs[n];
  T v = zero_of<T>();
  bool have = false;
  if (a.X1) {
    const T* x = static_cast<const T*>(a.X1) + base;
    T acc = mul(x[i], s1[0 + R * c]);
    for (int k = 1; k < R; ++k) fma_acc(acc, x[i + I * k], s1[k + R * c]);
    v = a.neg1 ? neg(acc) : acc;
    have = true;
  }
  if (a.X3) {
    const double cf = a.coef3_mu ? st->mu : a.coef3;
    T t = scale(static_cast<const T*>(a.X3)[base + idx], cf);
    v = have ? add(v, t) : t;
    have = true;
  }
  if (a.X2) {
    const T* x = static_cast<const T*>(a.X2) + base;
    T acc = mul(x[i], s2[0 + R * c]);
    for (int k = 1; k < R; ++k) fma_acc(acc, x[i + I * k], s2[k + R * c]);
    v = have ? add(v, acc) : acc;
    have = true;
  }
  if (a.X4) {
    T t = scale(static_cast<const T*>(a.X4)[base + idx], a.coef4);
    v = have ? add(v, t) : t;
  }
  static_cast<T*>(a.out)[base + idx] = v;
}

// Elementwise on stacked vectors: out = alpha*x + beta*y   (length n)
template <class T>
__global__ void k_axpby(const T* __restrict__ x, double alpha, const T* __restrict__ y, double beta, T* __restrict__ out,
                        int64_t n, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T v = scale(x[i], alpha);
  if (y) v = (beta == 1.0) ? add(v, y[i]) : (beta == -1.0 ? sub(v, y[i]) : add(v, scale(y[i], beta)));
  out[i] = v;
}

// ------------------------------------------------------------------------------------------
// Core-sized R x R kernels (one block per mode)
// ------------------------------------------------------------------------------------------
// w_n = W1_n - (C_n Gamma_n^T) Gti_n       (solver.py:134-137), written as vec into w (NR^2)
// E_n = I - (F_n + Gamma_n^T) Gti_n        (solver.py:181-184)
// Yg_n = Y_n Gti_n                         (hessian.py:346)
// S_n = sum_{m != n} (Gamma^(n,m) o Wm)^T  (hessian.py:318-325)
enum SmallOp : int { kOpW = 0, kOpE = 1, kOpYG = 2, kOpS = 3 };

template <class T>
__global__ void k_small(int op, const T* __restrict__ P0, const T* __restrict__ P1, const T* __restrict__ excl,
                        const T* __restrict__ Gti, const T* __restrict__ pair, int N, int R, T* __restrict__ out,
                        const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R2 = R * R;
  T* t0 = reinterpret_cast<T*>(smem_raw);
  T* t1 = t0 + R2;
  const int n = blockIdx.x;
  const T* gx = excl + (int64_t)n * R2;
  const T* gti = Gti + (int64_t)n * R2;
  if (op == kOpW) {
    // t0 = C_n @ Gamma_n^T
    const T* cn = P1 + (int64_t)n * R2;
    for (int e = threadIdx.x; e < R2; e += blockDim.x) {
      int i = e % R, j = e / R;
      T acc = mul(cn[i], gx[j]);  // (Gamma^T)[0, j] = Gamma[j, 0]
      for (int k = 1; k < R; ++k) fma_acc(acc, cn[i + R * k], gx[j + R * k]);
      t0[e] = acc;
    }
    __syncthreads();
    const T* w1 = P0 + (int64_t)n * R2;
    for (int e = threadIdx.x; e < R2; e += blockDim.x) {
      int i = e % R, j = e / R;
      T acc = mul(t0[i], gti[R * j]);
      for (int k = 1; k < R; ++k) fma_acc(acc, t0[i + R * k], gti[k + R * j]);
      out[(int64_t)n * R2 + e] = sub(w1[e], acc);
    }
  } else if (op == kOpE) {
    const T* fn = P0 + (int64_t)n * R2;
    for (int e = threadIdx.x; e < R2; e += blockDim.x) {
      int i = e % R, j = e / R;
      t0[e] = add(fn[e], gx[j + R * i]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R2; e += blockDim.x) {
      int i = e % R, j = e / R;
      T acc = mul(t0[i], gti[R * j]);
      for (int k = 1; k < R; ++k) fma_acc(acc, t0[i + R * k], gti[k + R * j]);
      out[(int64_t)n * R2 + e] = sub(from_real<T>(i == j ? 1.0 : 0.0), acc);
    }
  } else if (op == kOpYG) {
    const T* yn = P0 + (int64_t)n * R2;
    for (int e = threadIdx.x; e < R2; e += blockDim.x) {
      int i = e % R, j = e / R;
      T acc = mul(yn[i], gti[R * j]);
      for (int k = 1; k < R; ++k) fma_acc(acc, yn[i + R * k], gti[k + R * j]);
      out[(int64_t)n * R2 + e] = acc;
    }
  } else {  // kOpS
    for (int e = threadIdx.x; e < R2; e += blockDim.x) {
      int i = e % R, j = e / R;
      T acc = zero_of<T>();
      bool first = true;
      for (int m = 0; m < N; ++m) {
        if (m == n) continue;
        // (pair o W_m)^T [i, j] = pair[j, i] * W_m[j, i]
        const T* pm = pair + ((int64_t)n * N + m) * R2;
        const T* wm = P0 + (int64_t)m * R2;
        T v = mul(pm[j + R * i], wm[j + R * i]);
        acc = first ? v : add(acc, v);
        first = false;
      }
      out[(int64_t)n * R2 + e] = acc;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Normalisation (kruskal.py:170-198 equal energy; 201-214 unit modes for mu0)
// ------------------------------------------------------------------------------------------
// norms[n*R + r] = ||X_n[:, r]||_2
template <class T>
__global__ void k_colnorms(const T* __restrict__ X, Modes md, double* __restrict__ norms, const LmDeviceState* st,
                           const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  __shared__ double scratch[32];
  const int n = blockIdx.y, r = blockIdx.x;
  const int64_t I = md.dims[n];
  const T* x = X + md.offs[n] + I * r;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < I; i += blockDim.x) acc += abs2(x[i]);
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) norms[n * md.R + r] = sqrt(acc);
}

// Per column r: scale_n = target / norm_n, target = (prod_n norm_n)^(1/N); phase of the
// argmax-|.| entry of the scaled mode-1 column folded into mode N.  One block per column.
// mode 0 (preamble): a zero-norm column is an error (ZeroDivisionError, kruskal.py:184-185).
// mode 1 (trial candidate): the column is copied unscaled and st->cand_zero is raised; the
// reference only normalises accepted candidates, so k_decide turns it into an error on accept.
template <class T>
__global__ void k_normalize(const T* __restrict__ X, Modes md, const double* __restrict__ norms, T* __restrict__ out,
                            LmDeviceState* st, const DevFlags* fl, int gate, int mode) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  __shared__ double sval[32];
  __shared__ long long sidx[32];
  __shared__ double s_scale[kMaxModes];
  __shared__ T s_phase;
  __shared__ int s_bad;
  const int r = blockIdx.x, N = md.N, R = md.R;
  if (threadIdx.x == 0) {
    s_bad = 0;
    double prod = 1.0;
    for (int n = 0; n < N; ++n) {
      double v = norms[n * R + r];
      if (v == 0.0) s_bad = 1;
      prod = (n == 0) ? v : prod * v;
    }
    double target = pow(prod, 1.0 / N);
    for (int n = 0; n < N; ++n) s_scale[n] = target / norms[n * R + r];
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) {
      if (mode == 0) {
        if (st->err_code == 0) st->err_code = kErrZeroColumn;
      } else {
        st->cand_zero = 1;
      }
    }
    if (mode == 1)
      for (int n = 0; n < N; ++n) {
        const int64_t I = md.dims[n];
        for (int64_t i = threadIdx.x; i < I; i += blockDim.x) out[md.offs[n] + I * r + i] = X[md.offs[n] + I * r + i];
      }
    return;
  }
  // argmax over the scaled mode-1 column, first index on ties (np.argmax)
  const int64_t I0 = md.dims[0];
  const T* x0 = X + md.offs[0] + I0 * r;
  double best = -1.0;
  long long bi = 0;
  for (int64_t i = threadIdx.x; i < I0; i += blockDim.x) {
    double v = modulus(scale(x0[i], s_scale[0]));
    if (v > best) { best = v; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, best, o);
    long long oi = __shfl_down_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) { sval[wid] = best; sidx[wid] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = sval[0];
    long long ib = sidx[0];
    for (int w = 1; w < nw; ++w)
      if (sval[w] > b || (sval[w] == b && sidx[w] < ib)) { b = sval[w]; ib = sidx[w]; }
    T top = scale(x0[ib], s_scale[0]);
    double mag = modulus(top);
    s_phase = (mag != 0.0) ? dvd(top, from_real<T>(mag)) : from_real<T>(1.0);
  }
  __syncthreads();
  const T ph = s_phase;
  for (int n = 0; n < N; ++n) {
    const int64_t I = md.dims[n];
    const T* x = X + md.offs[n] + I * r;
    T* y = out + md.offs[n] + I * r;
    for (int64_t i = threadIdx.x; i < I; i += blockDim.x) {
      T v = scale(x[i], s_scale[n]);
      if (n == 0) v = dvd(v, ph);
      if (n == N - 1) v = mul(v, ph);
      y[i] = v;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Scalar reductions
// ------------------------------------------------------------------------------------------
// xx = sum_{r,s} Re prod_n C_n[r,s]  (||X||^2 from the Grams)
template <class T>
__global__ void k_xnorm2(const T* __restrict__ Cg, int N, int R, double* __restrict__ outp, const LmDeviceState* st,
                         const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  __shared__ double scratch[32];
  const int R2 = R * R;
  double acc = 0.0;
  for (int e = threadIdx.x; e < R2; e += blockDim.x) {
    T v = Cg[e];
    for (int n = 1; n < N; ++n) v = mul(v, Cg[(int64_t)n * R2 + e]);
    acc += re(v);
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) *outp = acc;
}

// Re sum conj(a_i) * b_i (+ mu * |a_i|^2 when with_mu: Re vdot(delta, g + mu*delta), solver.py:260)
template <class T>
__global__ void k_redot(const T* __restrict__ a, const T* __restrict__ b, int64_t n, int with_mu,
                        double* __restrict__ outp, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  __shared__ double scratch[32];
  const double mu = st->mu;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    T bi = b[i];
    if (with_mu) bi = add(bi, scale(a[i], mu));
    acc += re(a[i]) * re(bi) + im(a[i]) * im(bi);
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) *outp = acc;
}

// ||Y||^2 partials over a large buffer: grid-stride, per-block partial (fixed order)
template <class T>
__global__ void k_sumsq_partial(const T* __restrict__ y, int64_t n, double* __restrict__ part) {
  pdl_wait();
  __shared__ double scratch[32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += abs2(ld_stream(y + i));
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_sum_partials(const double* __restrict__ part, int n, double* __restrict__ outp,
                               const LmDeviceState* st = nullptr, const DevFlags* fl = nullptr, int gate = 0) {
  pdl_wait();
  if (gate && !gate_open(st, fl, gate)) return;
  __shared__ double scratch[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) *outp = acc;
}

// gated copy (commit of an accepted candidate, scatter of pass outputs)
template <class T>
__global__ void k_copy(const T* __restrict__ src, T* __restrict__ dst, int64_t n, const LmDeviceState* st,
                       const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

// 2-D gated copy: dst[r * ldd + i] = src[r * lds + i], i < rows, r < cols
template <class T>
__global__ void k_copy2d(const T* __restrict__ src, int64_t lds, T* __restrict__ dst, int64_t ldd, int64_t rows,
                         int64_t cols, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  int64_t i = idx % rows, r = idx / rows;
  dst[r * ldd + i] = src[r * lds + i];
}

__global__ void k_clear_pending(DevFlags* fl) {
  pdl_wait(); fl->pending_accept = 0; }

// Speculative rejection branch (engine.cu): mu of the branch = mu * growth, exactly k_decide's
// rho <= 0 update; its error flags are cleared first.  Launched on the main stream BEFORE the
// branch forks off, so the snapshot is stream-ordered ahead of this iteration's k_decide.
__global__ void k_spec_begin(LmDeviceState* st, double* mu_rej, int* sing) {
  pdl_wait();
  *mu_rej = st->mu * st->growth;
  *sing = 0;
  st->spec_iter = st->iter;
}
// After a rejection, the speculative branch's errors become the fit's (as the core system of a
// rejected step would have reported them at the end of that step)
__global__ void k_spec_errors(LmDeviceState* st, const DevFlags* fl, const int* sing, const int* info) {
  pdl_wait();
  if (!gate_open(st, fl, kOnRejectPrev)) return;
  if (*sing) st->err_code = kErrSingular;
  else if (*info != 0) st->err_code = st->use_kinv ? kErrSingular : kErrPhi1Singular;
}

// Guard band: the identity ||Y||^2 - 2Re<Y,X> + ||X||^2 has an absolute error of a
// few eps * ||Y||^2.  When the accept decision is within that band of a tie, or the residual is
// so small that the identity cannot resolve it (exact-fit problems), the candidate's residual --
// and, once, the current model's -- is recomputed directly from Y (k_direct_resid).
__global__ void k_precheck(const LmDeviceState* st, DevFlags* fl, const double* scal) {
  pdl_wait();
  if (st->stopped || st->err_code) {
    fl->need_direct = 0;
    fl->need_cur_direct = 0;
    return;
  }
  const double yx = scal[0], xx = scal[2];
  const double cs = st->ynorm_sq - 2.0 * yx + xx;
  const double scale_ = st->ynorm_sq + fabs(xx) + 2.0 * fabs(yx);
  const bool tiny = cs < 1e-10 * st->ynorm_sq;
  const bool close = fabs(st->err_sq - cs) <= 1e-12 * scale_;
  fl->need_direct = (tiny || close || st->force_direct) ? 1 : 0;
  fl->need_cur_direct = (fl->need_direct && !st->err_direct) ? 1 : 0;
}

// One LM decision (solver.py:354-383): trial error from the identity
//   ||Y - X||^2 = ||Y||^2 - 2 Re<Y,X> + ||X||^2,
// gain ratio (solver.py:259-263), Nielsen update (solver.py:238-248), accept test, trace record,
// tolerance window and mu overflow.  scal[0] = Re<Y,X_cand>, scal[2] = ||X_cand||^2,
// scal[3] = Re vdot(delta, g + mu delta).
__global__ void k_decide(LmDeviceState* st, DevFlags* fl, IterRecordDev* trace, const double* scal) {
  pdl_wait();
  if (st->stopped) return;
  const int t = st->iter + 1;
  if (st->err_code) {
    st->stopped = 3;
    st->err_iter = t;
    return;
  }
  const double yx = scal[0], xx = scal[2];
  const double denom = (t == st->test_negdenom_iter) ? -scal[3] : scal[3];
  const bool direct = fl->need_direct != 0;
  if (fl->need_cur_direct) {  // re-anchor the current error on a direct residual (kruskal.py:159-167)
    const double e0 = sqrt(scal[5]) / st->ynorm;
    const double es = e0 * st->ynorm;
    st->err = e0;
    st->err_sq = es * es;
    st->err_direct = 1;
  }
  fl->need_direct = 0;
  fl->need_cur_direct = 0;
  const double raw = direct ? scal[4] : st->ynorm_sq - 2.0 * yx + xx;
  const double cand_err = sqrt(fmax(raw, 0.0)) / st->ynorm;
  const double cs = cand_err * st->ynorm;
  const double cand_sq = cs * cs;
  double rho;
  if (fabs(denom) < 1e-30) rho = -1.0;
  else rho = (st->err_sq - cand_sq) / denom;
  double mu = st->mu, growth = st->growth;
  int ok;
  if (rho > 0) {
    const double q = 2.0 * rho - 1.0;
    mu = mu * fmax(1.0 / 3.0, 1.0 - q * q * q);
    growth = 2.0;
    ok = 1;
  } else {
    mu = mu * growth;
    growth = 2.0 * growth;
    ok = 0;
  }
  st->mu = mu;
  st->growth = growth;
  st->cand_err = cand_err;
  st->cand_sq = cand_sq;
  st->rho = rho;
  st->denom = denom;
  st->yx_re = yx;
  st->xx = xx;
  double d;
  int acc;
  if (ok && cand_err < st->err) {
    if (st->cand_zero) {  // normalize_equal_energy(candidate) raises ZeroDivisionError
      st->err_code = kErrZeroColumn;
      st->stopped = 3;
      st->err_iter = t;
      st->cand_zero = 0;
      return;
    }
    d = fabs(st->err - cand_err);
    st->err = cand_err;
    st->err_sq = cand_sq;
    st->err_direct = direct ? 1 : 0;
    acc = 1;
    fl->pending_accept = 1;
  } else {
    d = 0.0;
    acc = 0;
  }
  st->cand_zero = 0;
  st->accepted = acc;
  st->accept_iter = acc ? t : -1;
  st->rej_grow = ok ? 0 : 1;
  st->deltas[st->ndeltas % 10] = d;
  st->ndeltas += 1;
  trace[t - 1].relerr = st->err;
  trace[t - 1].mu = mu;
  trace[t - 1].iter = t;
  trace[t - 1].accepted = acc;
  st->iter = t;
  bool tol_stop = false;
  if (st->ndeltas >= 10) {
    tol_stop = true;
    for (int k = 0; k < 10; ++k)
      if (!(st->deltas[k] < st->tol)) tol_stop = false;
  }
  if (tol_stop) st->stopped = 1;
  else if (mu > 1e30) st->stopped = 2;
  else if (t >= st->max_iters) st->stopped = 4;
}

}  // namespace cpf
