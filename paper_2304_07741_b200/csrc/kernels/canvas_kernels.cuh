// Hand-written sm_100a kernel templates of the Canvas executor.
//
// Every device kernel the executor launches is one of these templates,
// instantiated with a *functor* that the lowering (paper_2304_07741_b200/
// lowering.py) emits for one concrete kernel graph: the functor evaluates the
// producer chain of one materialised tensor at one coordinate, with all
// rearrangements (Group / Shift / Unfold, App. A.1-A.3) and pointwise ops
// (ew / bcast, A.5, A.8) folded into its loads as index arithmetic with
// compile-time extents.  The templates own the thread mapping, tiling,
// shared-memory staging and reduction order:
//
//   pointwise<F>        one output element (or one softmax / fold row) per
//                       thread, grid-stride, coalesced along the innermost
//                       spatial dim
//   gemm_nk<F>          C[n][m][s] = sum_k A(m,k) B(n,k,s): FC forward and
//                       dgrad with a computed B operand (K3, SIMT path)
//   gemm_wgrad<F>       partial dW over a fixed chunk of (n,s) rows, then
//   reduce_partials<F>  an ordered sum of the partials -> deterministic wgrad
//
// The file is self-contained (no system headers) so NVRTC can compile it at
// plan creation; __graft_entry__.build() also compiles it with nvcc for
// sm_100a against a sample functor as the build check.
#pragma once

#ifndef INFINITY
#define INFINITY __int_as_float(0x7f800000)
#endif

#define CANVAS_MAX_KSLOTS 24

struct CanvasArgs {
  float* p[CANVAS_MAX_KSLOTS];  // tensors this launch touches (plan slot table)
  long long n;                   // images in the batch
  int beta;                      // 1: accumulate into the destination (Fig.-2 copies)
  int copy;                      // replica index (informational)
};

namespace canvas {

// ---------------------------------------------------------------------------
// K1/K2: pointwise maps, folds and softmax rows
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void pointwise(const CanvasArgs& a) {
  const long long total = a.n * F::PER;
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += step) {
    const long long n = i / F::PER;
    const int r = (int)(i - n * F::PER);
    F::run(a, n, r);
  }
}

// ---------------------------------------------------------------------------
// K3 (SIMT): FC forward / dgrad.  Rows t = n*S + s are flattened so small
// spatial extents (7x7) still fill 64-wide tiles.  B is evaluated by the
// functor (fused producer chain), staged through shared memory once per tile.
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void gemm_nk(const CanvasArgs& a) {
  constexpr int BM = 64, BT = 64, BK = 16;
  __shared__ float As[BK][BM];
  __shared__ float Bs[BK][BT];
  const long long T = a.n * (long long)F::S;
  const long long t0 = (long long)blockIdx.x * BT;
  const int m0 = blockIdx.y * BM;
  const int tid = threadIdx.x;
  const int lt = tid & 63, lk = tid >> 6;
  const long long tl = t0 + lt;
  const bool tl_ok = tl < T;
  const long long ln = tl_ok ? tl / F::S : 0;
  const int ls = tl_ok ? (int)(tl - ln * F::S) : 0;
  const int lm = m0 + lt;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < F::K; k0 += BK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int kk = lk + 4 * q;
      const int k = k0 + kk;
      As[kk][lt] = (lm < F::M && k < F::K) ? F::A(a, lm, k) : 0.f;
      Bs[kk][lt] = (tl_ok && k < F::K) ? F::B(a, ln, k, ls) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long long t = t0 + tx + 16 * j;
    if (t >= T) continue;
    const long long n = t / F::S;
    const int s = (int)(t - n * F::S);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m < F::M) F::store(a, n, m, s, acc[i][j]);
    }
  }
}

// ---------------------------------------------------------------------------
// K3 (SIMT): wgrad partials.  Block z reduces rows [z*TCHUNK, (z+1)*TCHUNK) of
// the (n,s) axis into P[z][m][j]; reduce_partials sums z in order.  No atomics:
// identical inputs give identical bits (SURVEY §7 decision 5).
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void gemm_wgrad(const CanvasArgs& a) {
  constexpr int BM = 64, BJ = 64, BT = 16;
  __shared__ float As[BT][BM + 1];
  __shared__ float Bs[BT][BJ + 1];
  const long long T = a.n * (long long)F::S;
  const int j0 = blockIdx.x * BJ, m0 = blockIdx.y * BM;
  const long long tbeg = (long long)blockIdx.z * F::TCHUNK;
  const long long tend = tbeg + F::TCHUNK < T ? tbeg + F::TCHUNK : T;
  const int tid = threadIdx.x;
  const int lt = tid & 15, lr = tid >> 4;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (long long t0 = tbeg; t0 < tend; t0 += BT) {
    const long long t = t0 + lt;
    const bool ok = t < tend;
    const long long n = ok ? t / F::S : 0;
    const int s = ok ? (int)(t - n * F::S) : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = lr + 16 * q;
      const int m = m0 + r, j = j0 + r;
      As[lt][r] = (ok && m < F::M) ? F::A(a, n, m, s) : 0.f;
      Bs[lt][r] = (ok && j < F::J) ? F::B(a, n, j, s) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int tt = 0; tt < BT; ++tt) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[tt][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[tt][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* P = F::partials(a) + (long long)blockIdx.z * F::M * F::J;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= F::M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int jj = j0 + tx + 16 * j;
      if (jj < F::J) P[(long long)m * F::J + jj] = acc[i][j];
    }
  }
}

template <class F>
__device__ __forceinline__ void reduce_partials(const CanvasArgs& a) {
  const long long T = a.n * (long long)F::S;
  const int Z = (int)((T + F::TCHUNK - 1) / F::TCHUNK);
  const float* __restrict__ P = a.p[0];
  float* __restrict__ out = a.p[1];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < F::MJ; idx += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < Z; ++z) s += P[(long long)z * F::MJ + idx];
    out[idx] = s;
  }
}

}  // namespace canvas
