// TEST INFRASTRUCTURE ONLY: host (g++) emulation of csrc/kernels/canvas_kernels.cuh.
//
// The lowering emits CUDA functors; compiling them against this header on
// the CPU lets the CPU test-suite check the *generated* index maps, adjoint
// gathers and launch schedule against the oracle without a GPU.  The
// templates here are plain sequential loops with the same reduction order as
// the device templates where it matters (wgrad partial chunks); the device
// tiling itself is checked by the GPU parity tests.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#define __device__
#define __global__
#define __forceinline__ inline
#define __launch_bounds__(...)
#define __restrict__
using std::max;
using std::min;
template <class T>
inline T __ldg(const T* p) { return *p; }
inline float __int_as_float(int i) {
  float f;
  std::memcpy(&f, &i, 4);
  return f;
}
inline int __float_as_int(float f) {
  int i;
  std::memcpy(&i, &f, 4);
  return i;
}
inline float __fadd_rn(float a, float b) { return a + b; }
inline float __fsub_rn(float a, float b) { return a - b; }
inline float __fmul_rn(float a, float b) { return a * b; }
struct float4 {
  float x, y, z, w;
};
inline float4 make_float4(float x, float y, float z, float w) { return float4{x, y, z, w}; }
namespace canvas {
inline float4 win4(const float4 a, const float4 b, const int m) {
  if (m == 0) return a;
  if (m == 1) return make_float4(a.y, a.z, a.w, b.x);
  if (m == 2) return make_float4(a.z, a.w, b.x, b.y);
  return make_float4(a.w, b.x, b.y, b.z);
}
}  // namespace canvas

#define CANVAS_MAX_KSLOTS 24
struct CanvasArgs {
  float* p[CANVAS_MAX_KSLOTS];
  long long n;
  int beta;
  int copy;
};

namespace canvas {
inline float* ptr_add(float* p, int off) { return p + off; }
inline float ldg_v(const float* p) { return *p; }
inline float ldg_vp(const float* p, bool c) { return c ? *p : 0.f; }
template <class F, int V = 1>
void pointwise(const CanvasArgs& a) {
  for (long long n = 0; n < a.n; ++n)
    for (int r = 0; r < (int)F::PER; ++r) F::run(a, n, r);
}

template <class F, int KS>
void pointwise_ks(const CanvasArgs& a) {
  for (long long n = 0; n < a.n; ++n)
    for (int r = 0; r < (int)F::PER; ++r) {
      float tot[F::NACC] = {};
      for (int p = 0; p < KS; ++p) {
        float acc[F::NACC];
        F::part(a, n, r, p, acc);
        for (int j = 0; j < F::NACC; ++j) tot[j] += acc[j];
      }
      F::put(a, n, r, tot);
    }
}

template <class F>
void pointwise_planes(const CanvasArgs& a) {
  for (long long n = 0; n < a.n; ++n)
    for (int q = 0; q < F::Q; ++q)
      for (int s = 0; s < F::S; ++s) F::run(a, n, q, s);
}

template <class F>
void pointwise4(const CanvasArgs& a) {
  for (long long n = 0; n < a.n; ++n)
    for (int r = 0; r < (int)F::PER; r += 4) F::run4(a, n, r);
}

template <class F>
void pointwise_planes4(const CanvasArgs& a) {
  for (long long n = 0; n < a.n; ++n)
    for (int q = 0; q < F::Q; ++q)
      for (int s = 0; s < F::S; s += 4) F::run4(a, n, q, s);
}

template <class F>
void gemm_nk(const CanvasArgs& a) {
  const long long T = a.n * (long long)F::S;
  float* col = new float[F::K];
  for (long long t = 0; t < T; ++t) {
    const long long n = t / F::S;
    const int s = (int)(t - n * F::S);
    for (int k = 0; k < F::K; ++k) {
      col[k] = F::B(a, n, k, s);
      if constexpr (F::SAVE_B) F::save_b(a, n, k, s, col[k]);
    }
    for (int m = 0; m < F::M; ++m) {
      float acc = 0.f;
      for (int k = 0; k < F::K; ++k) acc = std::fma(F::A(a, m, k), col[k], acc);
      F::store(a, n, m, s, acc);
    }
  }
  delete[] col;
}

template <class F>
void gemm_wgrad(const CanvasArgs& a) {
  const long long T = a.n * (long long)F::S;
  const long long Z = (a.n * (long long)F::SP + F::TCHUNK - 1) / F::TCHUNK;  // reduce reads partials up to SP
  float* av = new float[F::M];
  float* bv = new float[F::J];
  for (long long z = 0; z < Z; ++z) {
    float* P = F::partials(a) + z * F::M * F::J;
    std::memset(P, 0, sizeof(float) * F::M * F::J);
    const long long te = std::min<long long>((z + 1) * F::TCHUNK, T);
    for (long long t = z * F::TCHUNK; t < te; ++t) {
      const long long n = t / F::S;
      const int s = (int)(t - n * F::S);
      for (int m = 0; m < F::M; ++m) av[m] = F::A(a, n, m, s);
      for (int j = 0; j < F::J; ++j) bv[j] = F::B(a, n, j, s);
      for (int m = 0; m < F::M; ++m)
        for (int j = 0; j < F::J; ++j) P[m * F::J + j] = std::fma(av[m], bv[j], P[m * F::J + j]);
    }
  }
  delete[] av;
  delete[] bv;
}

template <class F>
void wgrad_small(const CanvasArgs& a) { gemm_wgrad<F>(a); }
template <class F>
void wgrad_small_v(const CanvasArgs& a) { gemm_wgrad<F>(a); }

template <class F, int SL>
void softmax_rows(const CanvasArgs& a) {
  for (long long n = 0; n < a.n; ++n)
    for (int r = 0; r < (int)F::ROWS; ++r) {
      float m = -INFINITY, s = 0.f;
      for (int j = 0; j < F::SPAN; ++j) m = std::max(m, F::in(a, n, r, j));
      for (int j = 0; j < F::SPAN; ++j) s += std::exp(F::in(a, n, r, j) - m);
      for (int j = 0; j < F::SPAN; ++j) F::out(a, n, r, j, std::exp(F::in(a, n, r, j) - m) / s);
    }
}

template <class F, int SL>
void rowdot_rows(const CanvasArgs& a) {
  for (long long n = 0; n < a.n; ++n)
    for (int r = 0; r < (int)F::ROWS; ++r) {
      float d = 0.f;
      for (int j = 0; j < F::SPAN; ++j) d += F::term(a, n, r, j);
      F::put(a, n, r, d);
    }
}

template <class F>
void reduce_partials(const CanvasArgs& a) {
  const long long T = a.n * (long long)F::S;
  const int Z = (int)((T + F::TCHUNK - 1) / F::TCHUNK);
  for (int idx = 0; idx < F::MJ; ++idx) {
    float s = 0.f;
    for (int z = 0; z < Z; ++z) s += a.p[0][(long long)z * F::MJ + idx];
    a.p[1][F::TJ > 0 ? (idx % F::TJ) * (F::MJ / F::TJ) + idx / F::TJ : idx] = s;
  }
}
// 4-pixel operand functors (F::VEC): the tcgen05 producers call B4row/B4k
// (A4row/A4k) on pixel quads; the emulation evaluates the operands the same way
template <class F>
void gemm_nk_vec(const CanvasArgs& a) {
  const long long T = a.n * (long long)F::SP;  // padded pixel range (F::SP >= S)
  float* col = new float[4 * F::K];
  for (long long t = 0; t < T; t += 4) {
    const long long n = t / F::SP;
    const int s = (int)(t - n * F::SP);
    const int nv = std::min(4, F::S - s);  // pixels of the quad inside the image
    for (int k = 0; k < F::K; ++k) {
      const typename F::B4R R = F::B4row(a, k);
      F::B4k(a, R, n, s, col + 4 * k);
      if constexpr (F::SAVE_B)
        for (int e = 0; e < nv; ++e) F::save_b(a, n, k, s + e, col[4 * k + e]);
    }
    for (int e = 0; e < nv; ++e)
      for (int m = 0; m < F::M; ++m) {
        float acc = 0.f;
        for (int k = 0; k < F::K; ++k) acc = std::fma(F::A(a, m, k), col[4 * k + e], acc);
        F::store(a, n, m, s + e, acc);
      }
  }
  delete[] col;
}

template <class F>
void gemm_wgrad_vec(const CanvasArgs& a) {
  if constexpr (F::NQ)
    if (a.n % 4) {  // the device template falls back to the scalar producers
      gemm_wgrad<F>(a);
      return;
    }
  const long long T = a.n * (long long)F::SP;  // padded pixel range (F::SP >= S)
  const long long Z = (T + F::TCHUNK - 1) / F::TCHUNK;
  float* av = new float[4 * F::M];
  float* bv = new float[4 * F::J];
  for (long long z = 0; z < Z; ++z) {
    float* P = F::partials(a) + z * F::M * F::J;
    std::memset(P, 0, sizeof(float) * F::M * F::J);
    const long long te = std::min<long long>((z + 1) * F::TCHUNK, T);
    for (long long t = z * F::TCHUNK; t < te; t += 4) {
      long long n = t / F::SP;
      int s = (int)(t - n * F::SP);
      if constexpr (F::NQ) {  // entries pixel-major, quads of 4 images
        s = (int)(t / a.n);
        n = t - (long long)s * a.n;
      }
      for (int m = 0; m < F::M; ++m) {
        F::A4k(a, F::A4row(a, m), n, s, av + 4 * m);
        if constexpr (!F::NQ)  // padded pixels (F::SP > S) contribute zero, as on the device
          for (int e = 0; e < 4; ++e) av[4 * m + e] = s + e < F::S ? av[4 * m + e] : 0.f;
      }
      for (int j = 0; j < F::J; ++j) F::B4k(a, F::B4row(a, j), n, s, bv + 4 * j);
      for (int e = 0; e < 4; ++e)
        for (int m = 0; m < F::M; ++m)
          for (int j = 0; j < F::J; ++j) P[m * F::J + j] = std::fma(av[4 * m + e], bv[4 * j + e], P[m * F::J + j]);
    }
  }
  delete[] av;
  delete[] bv;
}

// dgrad with the broadcast-adjoint epilogue (F::EPI_BC): packed column
// col = ct*NT + m*JT + jj holds replica m of lhs index j = ct*JT + jj
template <class F>
void gemm_nk_epi_bc(const CanvasArgs& a) {
  const long long T = a.n * (long long)F::S;
  constexpr int NT = F::EPI_M * F::EPI_JT, L = F::M / F::EPI_M;
  float* col = new float[F::K];
  float* out = new float[F::M];
  for (long long t = 0; t < T; ++t) {
    const long long n = t / F::S;
    const int s = (int)(t - n * F::S);
    for (int k = 0; k < F::K; ++k) col[k] = F::B(a, n, k, s);
    for (int m = 0; m < F::M; ++m) {
      float acc = 0.f;
      for (int k = 0; k < F::K; ++k) acc = std::fma(F::A(a, m, k), col[k], acc);
      out[m] = acc;
    }
    const auto XL = F::epi_lhs_ctx(a, n, s);
    const auto XR = F::epi_rhs_ctx(a, n, s);
    const auto XT = F::epi_term_ctx(a, n, s);
    const auto XS = F::epi_store_l_ctx(a, n, s);
    for (int j = 0; j < L; ++j) {
      const float l = F::epi_lhs(a, XL, j);
      float dl = 0.f;
      for (int m = 0; m < F::EPI_M; ++m)
        dl += F::epi_term(a, XT, m, j, out[(j / F::EPI_JT) * NT + m * F::EPI_JT + j % F::EPI_JT], l, F::epi_rhs(a, XR, m, j), true);
      F::epi_store_l(a, XS, j, dl, true);
    }
  }
  delete[] col;
  delete[] out;
}

template <class F>
void gemm_nk_tc(const CanvasArgs& a) {
  if constexpr (F::EPI_BC) gemm_nk_epi_bc<F>(a);
  else if constexpr (F::VEC) gemm_nk_vec<F>(a);
  else gemm_nk<F>(a);
}
template <class F>
void gemm_wgrad_tc(const CanvasArgs& a) {
  if constexpr (F::VEC) gemm_wgrad_vec<F>(a);
  else gemm_wgrad<F>(a);
}

template <class F, int NT, int STAGES, bool PACKED, bool A_MN, int PW = 8, int NACC = 1>
void tc_gemm_pix(const CanvasArgs& a) { gemm_nk_tc<F>(a); }
template <class F, int NT>
void tc_pack_b(const CanvasArgs&) {}
template <class F, int NT, int STAGES, int NACC = 1, int PW = 8, bool UNROLL = false>
void tc_gemm_pix_tmema(const CanvasArgs& a) { gemm_nk<F>(a); }
template <class F, int NT, int STAGES, int PW, int EW>
void tc_gemm_pix_persistent(const CanvasArgs& a) { gemm_nk_tc<F>(a); }
template <class F, int NT, int STAGES, int PW = 8, int JG = 1>
void tc_gemm_wgrad(const CanvasArgs& a) { gemm_wgrad_tc<F>(a); }
}  // namespace canvas
