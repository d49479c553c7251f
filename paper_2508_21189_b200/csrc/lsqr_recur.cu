// LSQR recurrences on the device: one CTA runs the d-length updates and the Paige & Saunders scalar
// recurrences of sketch-and-precondition LSQR (the driver the reference's rand_nla.py builds its
// least-squares solve around; SciPy `lsqr` semantics, damp = 0) between two fused passes over A
// (sk_lsqr_step_f32_f64).  The host then only reads back 8 scalars per iteration for the stopping
// test, instead of the d-vector [A^T u, ||u||^2] plus two d x d products in NumPy — the GPU no longer
// idles while the host forms the next v (config 4: ~0.25 ms per iteration).
//
// Scaling: the step is always called with coefficient 1 (u_dev <- A v'' - u_dev), and v'' carries the
// factor: with u_dev = c u (u normalised) and v'' = (c / alpha) R^-1 v, the new u_dev equals
// (c / alpha) beta u_new, so c' = ||u_dev_new|| = sqrt(zb[d]) and beta = c' alpha / c.
#include <cuda_runtime.h>

#include "common.cuh"

namespace skb {
namespace {

constexpr int R_THREADS = 512;

// state: [0] alpha  [1] c (scale of u_dev)  [2] phibar  [3] rhobar  [4] anorm2  [5] ddnorm  [6] bnorm
//        [7] atol  [8] btol  [9] istop  [10] itn
// scal (out, this iteration): [0] itn  [1] istop  [2] r1norm  [3] arnorm  [4] test2  [5] acond  [6] test1
//        [7] beta
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // red reused between calls
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];  // fixed order: deterministic
  return s;
}

__global__ void __launch_bounds__(R_THREADS) lsqr_recur_kernel(int d, const double* __restrict__ rinv,
                                                              const double* __restrict__ rinvt,
                                                              const double* __restrict__ zb, double* v, double* w,
                                                              double* x, double* vnext, double* state,
                                                              double* scal) {
  __shared__ double zs[R_THREADS];
  __shared__ double vs[R_THREADS];
  __shared__ double red[R_THREADS / 32];
  const int t = threadIdx.x;
  if (state[9] != 0.0) return;  // stopped: later launches leave x and the state alone
  const double alpha = state[0], c = state[1];
  double phibar = state[2], rhobar = state[3], anorm2 = state[4], ddnorm = state[5];
  const double bnorm = state[6], atol = state[7], btol = state[8];
  if (t < d) zs[t] = zb[t];
  const double cn = sqrt(zb[d]);
  const double beta = (c > 0.0 && alpha > 0.0) ? cn * alpha / c : 0.0;
  __syncthreads();
  // v <- R^-T A^T u_new - beta v, alpha_new = ||v||
  const double vold = t < d ? v[t] : 0.0;
  double vn = vold;
  if (beta > 0.0) {
    double g = 0.0;
    if (t < d)
      for (int j = 0; j < d; ++j) g = fma(rinv[(size_t)j * d + t], zs[j], g);  // (R^-T z)[t], coalesced
    vn = t < d ? g / cn - beta * vold : 0.0;
    anorm2 += alpha * alpha + beta * beta;
  }
  double an = alpha;
  if (beta > 0.0) {
    an = sqrt(block_sum(vn * vn, red));
    if (an > 0.0) vn /= an;
  }
  // Givens rotation and the x, w updates (Paige & Saunders)
  const double rho = hypot(rhobar, beta);
  const double cs = rhobar / rho, sn = beta / rho;
  const double theta = sn * an;
  rhobar = -cs * an;
  const double phi = cs * phibar;
  phibar = sn * phibar;
  const double tau = sn * phi;
  const double wold = t < d ? w[t] : 0.0;
  ddnorm += block_sum(wold * wold, red) / (rho * rho);
  double xn = 0.0;
  if (t < d) {
    xn = x[t] + (phi / rho) * wold;
    x[t] = xn;
    w[t] = vn - (theta / rho) * wold;
    v[t] = vn;
    vs[t] = vn;
  }
  const double xnorm = sqrt(block_sum(xn * xn, red));  // (syncs: vs complete)
  // next step input v'' = (c' / alpha_new) R^-1 v_new (rinvt[j][t] = rinv[t][j]: coalesced)
  if (t < d) {
    double g = 0.0;
    for (int j = 0; j < d; ++j) g = fma(rinvt[(size_t)j * d + t], vs[j], g);
    vnext[t] = an > 0.0 ? (cn / an) * g : 0.0;
  }
  if (t == 0) {
    const double anorm = sqrt(anorm2);
    const double r1norm = phibar, arnorm = an * fabs(tau);
    const double test1 = bnorm > 0.0 ? r1norm / bnorm : 0.0;
    const double test2 = anorm * r1norm > 0.0 ? arnorm / (anorm * r1norm) : 0.0;
    double istop = 0.0;
    if (test2 <= atol)
      istop = 2.0;
    else if (btol > 0.0 && test1 <= btol + atol * anorm * xnorm / bnorm)
      istop = 1.0;
    const double itn = state[10] + 1.0;
    state[0] = an;
    state[1] = cn;
    state[2] = phibar;
    state[3] = rhobar;
    state[4] = anorm2;
    state[5] = ddnorm;
    state[9] = istop;
    state[10] = itn;
    scal[0] = itn;
    scal[1] = istop;
    scal[2] = r1norm;
    scal[3] = arnorm;
    scal[4] = test2;
    scal[5] = sqrt(anorm2) * sqrt(ddnorm);
    scal[6] = test1;
    scal[7] = beta;
  }
}

}  // namespace
}  // namespace skb

// One LSQR iteration's recurrences after sk_lsqr_step_f32_f64 (called with coefficient 1): reads
// zb = [A^T u_dev, ||u_dev||^2], updates v, w, x, the state and writes vnext (the next step's v'') and
// 8 scalars.  d <= 512; Rinv and RinvT are d x d row-major (R^-1 and its transpose).  A no-op once the
// state records a stop.  Deterministic (fixed-order reductions).
extern "C" int sk_lsqr_recur_f64(int64_t d, const double* Rinv, const double* RinvT, const double* zb, double* v,
                                 double* w, double* x, double* vnext, double* state, double* scal, void* stream) {
  using namespace skb;
  if (d < 1 || d > R_THREADS) return fail(SK_EINVAL, "sk_lsqr_recur_f64: d must be in [1, 512]");
  if (!Rinv || !RinvT || !zb || !v || !w || !x || !vnext || !state || !scal)
    return fail(SK_EINVAL, "sk_lsqr_recur_f64: null pointer");
  lsqr_recur_kernel<<<1, R_THREADS, 0, as_stream(stream)>>>((int)d, Rinv, RinvT, zb, v, w, x, vnext, state, scal);
  return check_launch("sk_lsqr_recur_f64");
}
