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
typedef unsigned char uint8_t;

struct CanvasArgs {
  float* p[CANVAS_MAX_KSLOTS];  // tensors this launch touches (plan slot table)
  long long n;                   // images in the batch
  int beta;                      // 1: accumulate into the destination (Fig.-2 copies)
  int copy;                      // replica index (informational)
};

namespace canvas {

// p + off as one mad.wide (32-bit signed offset scaled to the 64-bit pointer):
// opaque to the compiler, so a per-lane base pointer shared by many rows is not
// re-associated into per-element 32-bit adds + sign-extended 64-bit math
__device__ __forceinline__ float* ptr_add(float* p, int off) {
  float* r;
  asm("mad.wide.s32 %0, %1, 4, %2;" : "=l"(r) : "r"(off), "l"(p));
  return r;
}

// the 4 consecutive words starting at word m (0..3) of the 8-word window a ++ b
// (a quad at a run-time 4 B offset from its two aligned 16 B chunks)
__device__ __forceinline__ float4 win4(const float4 a, const float4 b, const int m) {
  if (m == 0) return a;
  if (m == 1) return make_float4(a.y, a.z, a.w, b.x);
  if (m == 2) return make_float4(a.z, a.w, b.x, b.y);
  return make_float4(a.w, b.x, b.y, b.z);
}

// warp index of this thread, through a shuffle so the compiler can prove it
// warp-uniform: the warp-role branches of the tcgen05 templates then stay
// uniform and producer index math / memory descriptors live on the uniform
// datapath (measured 2-4% on the layer1 dgrad / wgrad launches)
// non-coherent loads the compiler may not re-sequence (asm volatile): a functor that
// issues them first keeps all of them in flight (Lowerer.loads_first, CANVAS_ASM_LOADS)
__device__ __forceinline__ float ldg_v(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ldg_vp(const float* p, const bool c) {
  float v = 0.f;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.f32 %0, [%1];\n\t}" : "+f"(v) : "l"(p), "r"((int)c));
  return v;
}

__device__ __forceinline__ int warp_index() {
#ifdef CANVAS_NO_WARP_SHFL
  return threadIdx.x >> 5;
#else
  return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
#endif
}

// ---------------------------------------------------------------------------
// K1/K2: pointwise maps, folds and softmax rows
// ---------------------------------------------------------------------------
// V > 1: each thread evaluates V elements blockDim apart (every load instruction
// stays coalesced), giving V independent gathers per thread.
template <class F, int V = 1>
__device__ __forceinline__ void pointwise(const CanvasArgs& a) {
  const long long total = a.n * F::PER;
  const long long chunk = (long long)blockDim.x * V;
  for (long long base = (long long)blockIdx.x * chunk; base < total; base += (long long)gridDim.x * chunk) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const long long i = base + j * blockDim.x + threadIdx.x;
      if (i < total) {
        const long long n = i / F::PER;
        F::run(a, n, (int)(i - n * F::PER));
      }
    }
  }
}

// KS consecutive lanes per output element (few outputs, long reduction): F::part
// accumulates lane `part`'s share of the reduction (terms part, part + KS, ...), the
// KS partial sums are combined by a fixed xor-shuffle tree (deterministic) and the
// group's first lane stores.  The element loop is block-uniform, so every lane of a
// warp reaches the shuffles; lanes past the end evaluate a clamped element.
template <class F, int KS>
__device__ __forceinline__ void pointwise_ks(const CanvasArgs& a) {
  static_assert(KS >= 2 && KS <= 32 && (KS & (KS - 1)) == 0, "KS: power of 2 <= 32");
  const long long total = a.n * F::PER;
  const int part = threadIdx.x % KS;
  const long long per_block = blockDim.x / KS;
  for (long long base = (long long)blockIdx.x * per_block; base < total; base += (long long)gridDim.x * per_block) {
    const long long i = base + threadIdx.x / KS;
    const bool ok = i < total;
    const long long ic = ok ? i : total - 1;
    const long long n = ic / F::PER;
    const int r = (int)(ic - n * F::PER);
    float acc[F::NACC];
    F::part(a, n, r, part, acc);
#pragma unroll
    for (int j = 0; j < F::NACC; ++j)
#pragma unroll
      for (int o = KS / 2; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (ok && part == 0) F::put(a, n, r, acc);
  }
}

// Plane-major variant: blockIdx.y = (image, channel plane) — block-uniform, so the
// functor's channel index math (flat-channel decomposition, replica/tap
// indices) runs once per warp on the uniform datapath — and the threads of
// gridDim.x blocks walk the H*W pixels of that plane (coalesced).
// gridDim.y is capped (~64 CTAs per SM over the launch), so each CTA strides
// over planes: block turnover stays off the critical path and the per-CTA
// setup is amortised.
template <class F>
__device__ __forceinline__ void pointwise_planes(const CanvasArgs& a) {
  const long long planes = a.n * F::Q;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;  // x fastest: co-resident CTAs share planes
  for (long long pq = blockIdx.y; pq < planes; pq += gridDim.y) {
    const long long n = pq / F::Q;
    const int q = (int)(pq - n * F::Q);
    if (s < F::S) F::run(a, n, q, s);
  }
}

// 4-element variants: each thread evaluates the 4 consecutive elements r .. r+3
// (F::run4; PER, resp. S, is a multiple of 4 so a quad stays in one image /
// plane).  The functor computes the lane-invariant part of its index math
// (channel / tap decomposition, replica loop bounds, row offsets) once per quad
// and issues each lane-affine gather from one address with immediate offsets.
template <class F>
__device__ __forceinline__ void pointwise4(const CanvasArgs& a) {
  const long long total = a.n * F::PER;
  for (long long i = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x); i < total; i += 4LL * gridDim.x * blockDim.x) {
    const long long n = i / F::PER;
    F::run4(a, n, (int)(i - n * F::PER));
  }
}

template <class F>
__device__ __forceinline__ void pointwise_planes4(const CanvasArgs& a) {
  const long long planes = a.n * F::Q;
  const int s = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  for (long long pq = blockIdx.y; pq < planes; pq += gridDim.y) {
    const long long n = pq / F::Q;
    const int q = (int)(pq - n * F::Q);
    if (s < F::S) F::run4(a, n, q, s);
  }
}

// ---------------------------------------------------------------------------
// K2: softmax / row-dot over a channel span with SL threads per row.  When
// rows are few and long (ResNet stage 4: 49 pixels x 512 channels) a thread
// per row starves the GPU; here RPB = 256/SL rows per CTA, each row's span is
// split across SL threads (rows innermost: loads stay coalesced along pixels)
// and the partial max / sum / dot are combined in shared memory in a fixed
// order (deterministic).  F::in(a,n,r,j), F::out(a,n,r,j,y) (softmax) or
// F::term(a,n,r,j), F::put(a,n,r,v) (row-dot); F::ROWS rows of F::SPAN.
// ---------------------------------------------------------------------------
template <class F, int SL>
__device__ __forceinline__ void softmax_rows(const CanvasArgs& a) {
  constexpr int RPB = 256 / SL;
  __shared__ float red[SL][RPB + 1];
  const long long total = a.n * F::ROWS;
  const int tr = threadIdx.x % RPB, sl = threadIdx.x / RPB;
  for (long long rb = (long long)blockIdx.x * RPB; rb < total; rb += (long long)gridDim.x * RPB) {
    const long long row = rb + tr;
    const bool ok = row < total;
    const long long n = ok ? row / F::ROWS : 0;
    const int r = ok ? (int)(row - n * F::ROWS) : 0;
    // a thread's slice of the row (PT values) stays in registers when short, so
    // the row is read from memory once
    constexpr int PT = (F::SPAN + SL - 1) / SL;
    constexpr bool REG = PT <= 64;
    float xv[REG ? PT : 1];
    float m = -INFINITY, s = 0.f;
    auto online = [&](float x) {
      if (x > m) {
        s = s * expf(m - x) + 1.f;
        m = x;
      } else {
        s += expf(x - m);
      }
    };
    if (ok) {
      if constexpr (REG) {
#pragma unroll
        for (int q = 0; q < PT; ++q) {
          const int j = sl + q * SL;
          if (j < F::SPAN) {
            xv[q] = F::in(a, n, r, j);
            online(xv[q]);
          }
        }
      } else {
        for (int j = sl; j < F::SPAN; j += SL) online(F::in(a, n, r, j));
      }
    }
    red[sl][tr] = m;
    __syncthreads();
    float M = red[0][tr];
#pragma unroll
    for (int i = 1; i < SL; ++i) M = fmaxf(M, red[i][tr]);
    __syncthreads();
    red[sl][tr] = m == -INFINITY ? 0.f : s * expf(m - M);
    __syncthreads();
    float S = 0.f;
#pragma unroll
    for (int i = 0; i < SL; ++i) S += red[i][tr];
    __syncthreads();
    if (ok) {
      if constexpr (REG) {
#pragma unroll
        for (int q = 0; q < PT; ++q) {
          const int j = sl + q * SL;
          if (j < F::SPAN) F::out(a, n, r, j, expf(xv[q] - M) / S);
        }
      } else {
        for (int j = sl; j < F::SPAN; j += SL) F::out(a, n, r, j, expf(F::in(a, n, r, j) - M) / S);
      }
    }
  }
}

template <class F, int SL>
__device__ __forceinline__ void rowdot_rows(const CanvasArgs& a) {
  constexpr int RPB = 256 / SL;
  __shared__ float red[SL][RPB + 1];
  const long long total = a.n * F::ROWS;
  const int tr = threadIdx.x % RPB, sl = threadIdx.x / RPB;
  for (long long rb = (long long)blockIdx.x * RPB; rb < total; rb += (long long)gridDim.x * RPB) {
    const long long row = rb + tr;
    const bool ok = row < total;
    const long long n = ok ? row / F::ROWS : 0;
    const int r = ok ? (int)(row - n * F::ROWS) : 0;
    float acc = 0.f;
    if (ok)
      for (int j = sl; j < F::SPAN; j += SL) acc += F::term(a, n, r, j);
    red[sl][tr] = acc;
    __syncthreads();
    if (sl == 0 && ok) {
      float d = 0.f;
#pragma unroll
      for (int i = 0; i < SL; ++i) d += red[i][tr];
      F::put(a, n, r, d);
    }
    __syncthreads();
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

// ---------------------------------------------------------------------------
// wgrad for FCs with few output channels (M <= 16, e.g. fc(G)): a tensor tile
// would be >90% padding.  Each CTA stages 64-pixel tiles of both operands in
// shared memory (coalesced along pixels) and each thread accumulates one or
// more (m, j) outputs over its pixel chunk; partials are reduced in order.
// grid = (ceil(J/JT), 1, chunks), JT = 256 / M rounded down to a power of 2.
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void wgrad_small(const CanvasArgs& a) {
  // thread (j = tid % JT, pixel group pg = tid / JT) accumulates all M outputs of
  // row j over the tile pixels q = pg (mod PG): per pixel one Bs read, one
  // (vector) As read of the M gradients and M FMAs; the PG partial sums are
  // combined in a fixed order at the end (deterministic)
  constexpr int TP = 64;
  constexpr int JT = F::JT;
  constexpr int PG = 256 / JT;
  constexpr int M = F::M;
  constexpr int MP = (M + 3) / 4 * 4;
  __shared__ __align__(16) float As[TP][MP];
  __shared__ float Bs[JT][TP + 1];
  __shared__ float red[PG > 1 ? PG : 1][M][JT];
  const long long T = a.n * (long long)F::S;
  const long long tbeg = (long long)blockIdx.z * F::TCHUNK;
  const long long tend = tbeg + F::TCHUNK < T ? tbeg + F::TCHUNK : T;
  const int j0 = blockIdx.x * JT;
  const int tid = threadIdx.x;
  const int oj = tid % JT, pg = tid / JT;
  float acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = 0.f;
  for (long long t0 = tbeg; t0 < tend; t0 += TP) {
    const int p = tid % TP;
    const long long t = t0 + p;
    const bool ok = t < tend;
    const long long n = ok ? t / F::S : 0;
    const int s = ok ? (int)(t - n * F::S) : 0;
    for (int r = tid / TP; r < MP; r += blockDim.x / TP) As[p][r] = (ok && r < M) ? F::A(a, n, r < M ? r : 0, s) : 0.f;
    for (int r = tid / TP; r < JT; r += blockDim.x / TP) {
      const int j = j0 + r;
      Bs[r][p] = (ok && j < F::J) ? F::B(a, n, j, s) : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int q = pg; q < TP; q += PG) {
      const float b = Bs[oj][q];
#pragma unroll
      for (int m4 = 0; m4 < MP; m4 += 4) {
        const float4 av = *reinterpret_cast<const float4*>(&As[q][m4]);
        if (m4 + 0 < M) acc[m4 + 0] = fmaf(av.x, b, acc[m4 + 0]);
        if (m4 + 1 < M) acc[m4 + 1] = fmaf(av.y, b, acc[m4 + 1]);
        if (m4 + 2 < M) acc[m4 + 2] = fmaf(av.z, b, acc[m4 + 2]);
        if (m4 + 3 < M) acc[m4 + 3] = fmaf(av.w, b, acc[m4 + 3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < M; ++m) red[PG > 1 ? pg : 0][m][oj] = acc[m];
  __syncthreads();
  for (int o = tid; o < M * JT; o += blockDim.x) {
    const int m = o / JT, jj = o % JT;
    float v = 0.f;
#pragma unroll
    for (int g = 0; g < PG; ++g) v += red[g][m][jj];
    if (j0 + jj < F::J) F::partials(a)[((long long)blockIdx.z * M + m) * F::J + j0 + jj] = v;
  }
}

// wgrad for few output channels with the 4-pixel functors (F::VEC, S % 4 == 0):
// no shared-memory staging and one barrier per CTA.  Warp (jg, ps) keeps JW rows
// j of the J side and all M rows of the M side for its pixel quads in registers:
// per 128-pixel strip (lane = one quad) it evaluates the M quads once, then per
// row j one quad of B and 4·M FMAs into lane-private sums acc[j][m].  At the end
// of the chunk the lane sums are reduced by a fixed xor-shuffle tree, the WP
// pixel streams in order through shared memory (deterministic).  Strips of one
// stream are ps, ps + WP, ... so the streams of a CTA read adjacent lines.
// grid = (ceil(J / (WJ·JW)), 1, chunks).
template <class F>
__device__ __forceinline__ void wgrad_small_v(const CanvasArgs& a) {
  constexpr int M = F::M, JW = F::JW, WJ = F::WJ, WP = 8 / WJ;
  static_assert(WJ * WP == 8, "8 warps = j groups x pixel streams");
  __shared__ float red[WP > 1 ? WP : 1][WJ][JW * M];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jg = warp % WJ, ps = warp / WJ;
  const int jb = (blockIdx.x * WJ + jg) * JW;  // first row of this warp
  const long long T = a.n * (long long)F::S;
  const long long tbeg = (long long)blockIdx.z * F::TCHUNK;
  const long long tend = tbeg + F::TCHUNK < T ? tbeg + F::TCHUNK : T;
  typename F::A4R ra[M];
  typename F::B4R rb[JW];
#pragma unroll
  for (int m = 0; m < M; ++m) ra[m] = F::A4row(a, m);
#pragma unroll
  for (int j = 0; j < JW; ++j) rb[j] = F::B4row(a, jb + j < F::J ? jb + j : F::J - 1);
  float acc[JW][M];
#pragma unroll
  for (int j = 0; j < JW; ++j)
#pragma unroll
    for (int m = 0; m < M; ++m) acc[j][m] = 0.f;
  for (long long t = tbeg + 128 * ps + 4 * lane; t < tend; t += 128 * WP) {
    const long long n = t / F::S;
    const int s = (int)(t - n * F::S);
    float av[M][4];
#pragma unroll
    for (int m = 0; m < M; ++m) F::A4k(a, ra[m], n, s, av[m]);
#pragma unroll
    for (int j = 0; j < JW; ++j) {
      float bv[4];
      F::B4k(a, rb[j], n, s, bv);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        float v = acc[j][m];
#pragma unroll
        for (int e = 0; e < 4; ++e) v = fmaf(av[m][e], bv[e], v);
        acc[j][m] = v;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < JW; ++j)
#pragma unroll
    for (int m = 0; m < M; ++m) {
      float v = acc[j][m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (((j * M + m) & 31) == lane) red[WP > 1 ? ps : 0][jg][j * M + m] = v;
    }
  __syncthreads();
  float* P = F::partials(a) + (long long)blockIdx.z * M * F::J;
  for (int o = threadIdx.x; o < WJ * JW * M; o += blockDim.x) {
    const int g = o / (JW * M), r = o - g * (JW * M);
    const int j = (blockIdx.x * WJ + g) * JW + r / M, m = r % M;
    float v = 0.f;
#pragma unroll
    for (int p = 0; p < WP; ++p) v += red[p][g][r];
    if (j < F::J) P[(long long)m * F::J + j] = v;
  }
}

// F::TJ > 0: partials are [M][TJ] and dW is written transposed ([TJ][M]).
template <class F>
__device__ __forceinline__ int reduce_out_index(const int idx) {
  if constexpr (F::TJ > 0) return (idx % F::TJ) * (F::MJ / F::TJ) + idx / F::TJ;
  else return idx;
}

template <class F>
__device__ __forceinline__ void reduce_partials(const CanvasArgs& a) {
  const long long T = a.n * (long long)F::S;
  const int Z = (int)((T + F::TCHUNK - 1) / F::TCHUNK);
  const float* __restrict__ P = a.p[0];
  float* __restrict__ out = a.p[1];
  if (F::MJ >= 4096) {  // enough outputs: one thread per output, z in order
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < F::MJ; idx += gridDim.x * blockDim.x) {
      float s = 0.f;
      for (int z = 0; z < Z; ++z) s += P[(long long)z * F::MJ + idx];
      out[reduce_out_index<F>(idx)] = s;
    }
    return;
  }
  // few outputs: one warp per output, lane-strided z then a fixed shuffle tree
  const int lane = threadIdx.x & 31;
  for (int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < F::MJ; idx += (gridDim.x * blockDim.x) >> 5) {
    float s = 0.f;
    for (int z = lane; z < Z; z += 32) s += P[(long long)z * F::MJ + idx];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[reduce_out_index<F>(idx)] = s;
  }
}


// ===========================================================================
// K3 (tensor cores): tcgen05 3xTF32 GEMMs with a computed operand.
//
// The FC contraction runs on the 5th-gen tensor cores in split precision:
// x = hi + lo with hi = rna_tf32(x), lo = rna_tf32(x - hi), and
// D += A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in fp32 in TMEM, which
// meets fp32 tolerance where plain TF32 fails (SURVEY §7 decision 4).
//
// Warp roles (288 threads): warps 0-7 are producers — they evaluate the
// functor operands (the fused producer chain of the FC input: unfold /
// shift / group index maps and pointwise ops folded into the loads), split
// them, and store them into a STAGES-deep ring of 128B-swizzled K-major smem
// tiles (the canonical UMMA layout, 1024 B atoms); warp 8 allocates TMEM and
// one elected lane issues tcgen05.mma (M=128, N=NT, K=8 per instruction) and
// tcgen05.commit back to the producers; after the last k-block warps 0-7
// drain TMEM with tcgen05.ld (warp w reads lane quadrant w%4, column half w/4)
// and run the functor's store epilogue.
// ===========================================================================
typedef unsigned int cv_u32;
typedef unsigned long long cv_u64;

namespace tc {

__device__ __forceinline__ cv_u32 smem_u32(const void* p) {
  return (cv_u32)__cvta_generic_to_shared(p);
}
// 1024-aligned view of the dynamic smem window, derived by pointer arithmetic
// on the __shared__ array so the compiler keeps the shared address space
// (STS/LDS with 32-bit addresses instead of generic 64-bit stores)
__device__ __forceinline__ uint8_t* align_smem(uint8_t* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}
__device__ __forceinline__ void mbar_init(cv_u64* bar, cv_u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(cv_u64* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(cv_u64* bar, cv_u32 parity) {
  const cv_u32 a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity), "r"(0x989680)  // suspend-time hint: sleep instead of spinning on issue slots
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(cv_u64* bar, cv_u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// TMA bulk copy (1-D) global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, cv_u32 bytes, cv_u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// warm L2 with the 128 B line at p (the producers' upcoming gathers)
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// split x into (hi, lo) for 3xTF32: hi = x with the 13 low mantissa bits
// cleared (exactly a tf32 value), lo = x - hi (exact in fp32, |lo| < 2^-10 |x|),
// stored raw: the MMA consumes only lo's top 19 bits, an error below
// 2^-10 |lo| <= 2^-20 |x| per operand.  hi*hi + hi*lo + lo*hi then carries
// ~3 * 2^-20 relative error per product, two orders under the fp32 tolerance
// after fp32 accumulation (measured margin: worst element at 8% of
// 1e-5 + 1e-4|y| for K = 4608); 2 instructions per element (LOP3, FADD).
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
  lo = x - hi;
}

__device__ __forceinline__ void st_shared_v4(void* p, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// K-major, 128B-swizzle smem descriptor (rows of 128 B, 8-row atoms 1024 B apart)
__device__ __forceinline__ cv_u64 desc_k_sw128(cv_u32 saddr) {
  cv_u64 d = 0;
  d |= (cv_u64)((saddr >> 4) & 0x3FFF);
  d |= (cv_u64)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (cv_u64)(1024 >> 4) << 32;       // SBO: 8 rows x 128 B
  d |= (cv_u64)1 << 46;                 // descriptor version (sm_100)
  d |= (cv_u64)2 << 61;                 // SWIZZLE_128B
  return d;
}

// MN-major smem descriptor for 32-bit (tf32) operands: the only legal MN-major
// tf32 layout is SWIZZLE_128B_BASE32B — 128 B rows of 32 consecutive M
// elements, 4 K rows per 512 B atom, 32 B chunks XOR-permuted by row; M blocks
// of 32 are `lbo` bytes apart, K groups of 4 rows `sbo` bytes apart.
__device__ __forceinline__ cv_u64 desc_mn_sw128_32b(cv_u32 saddr, cv_u32 lbo, cv_u32 sbo) {
  cv_u64 d = 0;
  d |= (cv_u64)((saddr >> 4) & 0x3FFF);
  d |= (cv_u64)((lbo >> 4) & 0x3FFF) << 16;
  d |= (cv_u64)((sbo >> 4) & 0x3FFF) << 32;
  d |= (cv_u64)1 << 46;
  d |= (cv_u64)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}

// instruction descriptor: kind::tf32, D fp32, M=128, N=n; A K-major or MN-major, B K-major
__host__ __device__ constexpr cv_u32 idesc_tf32(int n, bool a_mn = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((cv_u32)(n >> 3) << 17) |
         ((cv_u32)(128 >> 4) << 24);
}

// byte offset of element (m, k) of a 128 x 32 MN-major SW128_BASE32B tile laid
// out as [k-group of 4 rows (8)][m-block of 32 (4)] atoms of 512 B
// (LBO = 512, SBO = 2048; one K=8 MMA spans two k-groups = 4096 B)
__device__ __forceinline__ int mn_off(int m, int k) {
  const int j = k & 3;
  return (((k >> 2) * 4 + (m >> 5)) << 9) + j * 128 + ((((m >> 3) & 3) ^ j) << 5) + (m & 7) * 4;
}

__device__ __forceinline__ void mma_tf32(cv_u32 dtmem, cv_u64 adesc, cv_u64 bdesc, cv_u32 idesc, cv_u32 accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

// A operand from tensor memory (K-major: TMEM lane = MMA row, one column per K
// element), B from shared memory
__device__ __forceinline__ void mma_tf32_ts(cv_u32 dtmem, cv_u32 atmem, cv_u64 bdesc, cv_u32 idesc, cv_u32 accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
      "r"(atmem), "l"(bdesc), "r"(idesc), "r"(accum));
}

// registers -> TMEM: 16 consecutive columns of this thread's lane (warp quadrant)
__device__ __forceinline__ void tmem_st16(cv_u32 taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st8(cv_u32 taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
               "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void commit(cv_u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(cv_u32* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_free(cv_u32 taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}

__device__ __forceinline__ void tmem_ld16(cv_u32 taddr, float* v) {
  cv_u32 r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void tmem_ld8(cv_u32 taddr, float* v) {
  cv_u32 r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void tmem_ld32(cv_u32 taddr, float* v) {
  cv_u32 r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

template <int N>
struct TmemCols {
  static constexpr int value = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : N <= 256 ? 256 : 512;
};

#ifndef CANVAS_WGRAD_STACK
#define CANVAS_WGRAD_STACK 1
#endif
constexpr bool WGRAD_STACK = CANVAS_WGRAD_STACK;  // stacked-N hi.hi + hi.lo wgrad MMA (wgrad_stack)
constexpr int kProducerWarps = 8;
constexpr int kThreads = (kProducerWarps + 2) * 32;  // + MMA warp + bulk-copy warp
constexpr int kBM = 128;  // MMA rows per tile
constexpr int kBK = 32;   // tf32 per 128 B swizzle row = one k-block

// swizzled byte offset of 16 B chunk c (0..7) of row r in a K-major SW128 tile
__device__ __forceinline__ int swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

// Shared memory plan of one pipeline: STAGES x {A_hi, A_lo, B_hi, B_lo} + barriers.
template <int NT, int STAGES>
struct Smem {
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int B_BYTES = NT * 128;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE;
  static constexpr int BYTES = BAR_OFF + (2 * STAGES + 1) * 8 + 16 + 1024;  // + alignment slack
};

// Shared memory plan of the wgrad pipeline with JG row tiles of 128 per CTA:
// STAGES x {A_hi[JG], A_lo[JG], B_hi, B_lo} + barriers.
template <int NT, int JG, int STAGES>
struct SmemW {
  static constexpr int A_TILE = kBM * 128;
  static constexpr int A_BYTES = JG * A_TILE;
  static constexpr int B_BYTES = NT * 128;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE;
  static constexpr int BYTES = BAR_OFF + (2 * STAGES + 1) * 8 + 16 + 1024;
};

// wgrad MMA issuer: per k-block, JG row tiles x 4 K=8 steps x 3 MMAs, tile g
// accumulating into TMEM columns [g*NT, (g+1)*NT)
// wgrad_stack<NT>(): with 2·NT <= 256 the hi.hi and hi.lo products are ONE MMA of
// N = 2·NT over the contiguous [B_hi; B_lo] rows (A_hi read from shared memory once
// instead of twice), accumulating into columns [0, NT) and [NT, 2·NT) of the tile's
// region; lo.hi adds into [0, NT); the epilogue sums the two halves
template <int NT>
__host__ __device__ constexpr bool wgrad_stack() { return WGRAD_STACK && 2 * NT <= 256; }

template <int NT, int JG, int STAGES>
__device__ __forceinline__ void mma_loop_w(uint8_t* smem, cv_u64* full, cv_u64* empty, cv_u64* done, cv_u32 tmem, int KB) {
  using L = SmemW<NT, JG, STAGES>;
  constexpr bool STACK = wgrad_stack<NT>();
  constexpr cv_u32 idesc = idesc_tf32(NT, false);
  constexpr cv_u32 idesc2 = idesc_tf32(STACK ? 2 * NT : NT, false);
  for (int kb = 0; kb < KB; ++kb) {
    const int st = kb % STAGES;
    mbar_wait(&full[st], (kb / STAGES) & 1);
    fence_after();
    const cv_u32 base = smem_u32(smem + st * L::STAGE);
    const cv_u32 b_hi = base + 2 * L::A_BYTES;
    const cv_u32 b_lo = b_hi + L::B_BYTES;
#pragma unroll
    for (int g = 0; g < JG; ++g) {
      const cv_u32 a_hi = base + g * L::A_TILE;
      const cv_u32 a_lo = a_hi + L::A_BYTES;
      const cv_u32 d = tmem + g * (STACK ? 2 * NT : NT);
#pragma unroll
      for (int kk = 0; kk < kBK / 8; ++kk) {
        const cv_u32 o = kk * 32;
        if constexpr (STACK) {
          mma_tf32(d, desc_k_sw128(a_hi + o), desc_k_sw128(b_hi + o), idesc2, !(kb == 0 && kk == 0));
          mma_tf32(d, desc_k_sw128(a_lo + o), desc_k_sw128(b_hi + o), idesc, 1);
        } else {
          mma_tf32(d, desc_k_sw128(a_hi + o), desc_k_sw128(b_hi + o), idesc, !(kb == 0 && kk == 0));
          mma_tf32(d, desc_k_sw128(a_hi + o), desc_k_sw128(b_lo + o), idesc, 1);
          mma_tf32(d, desc_k_sw128(a_lo + o), desc_k_sw128(b_hi + o), idesc, 1);
        }
      }
    }
    commit(&empty[st]);
  }
  commit(done);
}

// MMA issuer: consumes STAGES-deep ring, 3 MMAs per K=8 step (hi.hi, hi.lo, lo.hi)
// NACC > 1: the K loop is split into NACC contiguous chunks accumulated in
// separate TMEM regions (tmem + i*NT) and summed by the epilogue in fp32: the
// tensor core's accumulation error grows with the accumulated length, and
// chunking keeps K = 9C = 4608 (ResNet stage 4) inside the fp32 tolerance.
template <int NT, int STAGES, bool A_MN = false, int NACC = 1>
__device__ __forceinline__ void mma_loop(uint8_t* smem, cv_u64* full, cv_u64* empty, cv_u64* done, cv_u32 tmem, int KB) {
  using L = Smem<NT, STAGES>;
  constexpr cv_u32 idesc = idesc_tf32(NT, A_MN);
  for (int kb = 0; kb < KB; ++kb) {
    const int acc = (kb * NACC) / KB;
    const bool fresh = kb == 0 || ((kb - 1) * NACC) / KB != acc;
    const cv_u32 d = tmem + acc * NT;
    const int st = kb % STAGES;
    mbar_wait(&full[st], (kb / STAGES) & 1);
    fence_after();
    const cv_u32 a_hi = smem_u32(smem + st * L::STAGE);
    const cv_u32 a_lo = a_hi + L::A_BYTES;
    const cv_u32 b_hi = a_lo + L::A_BYTES;
    const cv_u32 b_lo = b_hi + L::B_BYTES;
#pragma unroll
    for (int kk = 0; kk < kBK / 8; ++kk) {
      const cv_u32 o = kk * 32;  // 8 tf32 = 32 B along K inside the swizzled row
      cv_u64 dah, dal;
      if (A_MN) {
        dah = desc_mn_sw128_32b(a_hi + kk * 4096, 512, 2048);
        dal = desc_mn_sw128_32b(a_lo + kk * 4096, 512, 2048);
      } else {
        dah = desc_k_sw128(a_hi + o);
        dal = desc_k_sw128(a_lo + o);
      }
      mma_tf32(d, dah, desc_k_sw128(b_hi + o), idesc, !(fresh && kk == 0));
      mma_tf32(d, dah, desc_k_sw128(b_lo + o), idesc, 1);
      mma_tf32(d, dal, desc_k_sw128(b_hi + o), idesc, 1);
    }
    commit(&empty[st]);
  }
  commit(done);
}

}  // namespace tc

// ---------------------------------------------------------------------------
// FC forward / dgrad on tensor cores: out[n][m][s] = sum_k A(m,k) B(n,k,s),
// MMA rows = 128 pixels t = n*S + s (operand B(n,k,s), computed), MMA cols =
// NT output channels (operand A(m,k), weights).
// ---------------------------------------------------------------------------
template <class F, int NT, int STAGES, bool PACKED, bool A_MN, int PW = tc::kProducerWarps, int NACC = 1>
__device__ __forceinline__ void tc_gemm_pix(const CanvasArgs& a) {
  static_assert(A_MN || PW == tc::kProducerWarps, "K-major producer mapping assumes 8 warps");
  static_assert(32 % PW == 0 && PW % 4 == 0, "PW must divide the k-block and cover the TMEM quadrants");
  using namespace tc;
  using L = Smem<NT, STAGES>;
  constexpr int NCOLS = TmemCols<NT * NACC>::value;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem(smem_raw);
  cv_u64* full = (cv_u64*)(smem + L::BAR_OFF);
  cv_u64* empty = full + STAGES;
  cv_u64* done = empty + STAGES;
  cv_u32* tslot = (cv_u32*)(done + 1);
  const int warp = warp_index(), lane = threadIdx.x & 31;
  constexpr int KB = (F::K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], PW * 32 + (PACKED ? 1 : 0));
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == PW) tmem_alloc<NCOLS>(tslot);
  fence_before();
  __syncthreads();
  fence_after();
  const cv_u32 tmem = *tslot;

  // SX: pixels per image of the GEMM's column space — F::SP (S rounded up to a
  // multiple of 4) for the quad producers, whose padding columns are not stored
  constexpr int SX = (A_MN && F::VEC) ? F::SP : F::S;
  const long long T = a.n * (long long)SX;
  const long long t0 = (long long)blockIdx.x * kBM;
  const int c0 = blockIdx.y * NT;

  if (warp < PW) {
    const int p = threadIdx.x;  // 0..255
    if constexpr (A_MN && F::VEC) {
      // MN-major A, 4-pixel functor: lane owns tile pixels 4*lane .. 4*lane+3 (one
      // 16 B chunk of a swizzled row), warp w owns k-rows w*ROWS .. (warp-uniform
      // row context).  The functor shares its index math and addresses across the
      // 4 pixels; stores are 16 B.  SX % 4 == 0, so a quad never straddles images.
      constexpr int ROWS = kBK / PW;
      const long long tq = t0 + 4 * lane;
      const bool okq = tq < T;
      const int pn = okq ? (int)(tq / SX) : 0;
      const int ps = okq ? (int)(tq - (long long)pn * SX) : 0;
      const int lm = SX != F::S ? (1 << (F::S - ps < 4 ? F::S - ps : 4)) - 1 : 15;  // lanes inside the image
      auto put = [&](int kb, float (&va)[ROWS][4]) {
        const int st = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
        uint8_t* sa_hi = smem + st * L::STAGE;
        uint8_t* sa_lo = sa_hi + L::A_BYTES;
#pragma unroll
        for (int q = 0; q < ROWS; ++q) {
          const int k = kb * kBK + warp * ROWS + q;
          const bool ok = okq && k < F::K;
          float h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool oke = ok && ((lm >> e) & 1);
            if constexpr (F::SAVE_B) {
              if (oke) F::save_b(a, (long long)pn, k, ps + e, va[q][e]);
            }
            split_tf32(oke ? va[q][e] : 0.f, h[e], l[e]);
          }
          const int off = mn_off(4 * lane, warp * ROWS + q);
          *reinterpret_cast<float4*>(sa_hi + off) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(sa_lo + off) = make_float4(l[0], l[1], l[2], l[3]);
        }
        fence_async_smem();
        mbar_arrive(&full[st]);
      };
      auto row = [&](int kb, int q) {
        const int k = kb * kBK + warp * ROWS + q;
        return F::B4row(a, k < F::K ? k : F::K - 1);
      };
      if constexpr (F::SPLIT) {
        // software pipeline: k-block kb+1's gathers are in flight while kb is combined and stored
        constexpr int NB = F::B4NRAW;
        float x0[ROWS][NB], x1[ROWS][NB];
        auto issue = [&](int kb, float (&x)[ROWS][NB]) {
#pragma unroll
          for (int q = 0; q < ROWS; ++q) F::B4ld(a, row(kb, q), (long long)pn, ps, x[q]);
        };
        auto commit_kb = [&](int kb, const float (&x)[ROWS][NB]) {
          float va[ROWS][4];
#pragma unroll
          for (int q = 0; q < ROWS; ++q) F::B4cp(a, row(kb, q), x[q], va[q]);
          put(kb, va);
        };
        issue(0, x0);
        for (int kb = 0; kb < KB; kb += 2) {
          if (kb + 1 < KB) issue(kb + 1, x1);
          commit_kb(kb, x0);
          if (kb + 1 < KB) {
            if (kb + 2 < KB) issue(kb + 2, x0);
            commit_kb(kb + 1, x1);
          }
        }
      } else {
        float va[ROWS][4];
        auto gather = [&](int kb) {
#pragma unroll
          for (int q = 0; q < ROWS; ++q) F::B4k(a, row(kb, q), (long long)pn, ps, va[q]);
        };
        gather(0);
        for (int kb = 0; kb < KB; ++kb) {
          put(kb, va);
          if (kb + 1 < KB) gather(kb + 1);
        }
      }
    } else {
    if (A_MN) {
      // MN-major A: warp w owns k-rows 4w..4w+3 of the 32-wide k-block, lane =
      // pixel within each 32-pixel block (4 blocks).  k is warp-uniform, so the
      // functor's channel index math runs once per k on the uniform datapath;
      // loads are 128 B coalesced; smem stores hit one 128 B swizzled row.
      int pn[4], ps[4];
      unsigned okmask = 0;
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) {
        const long long t = t0 + mb * 32 + lane;
        okmask |= (t < T ? 1u : 0u) << mb;
        const long long tc = t < T ? t : T - 1;
        pn[mb] = (int)(tc / F::S);
        ps[mb] = (int)(tc - (long long)pn[mb] * F::S);
      }
      // warm L2 with every source row of this CTA's 128-pixel tile (4 lines per row)
      if constexpr (F::NPF > 0) {
        for (int i = threadIdx.x; i < F::NPF * 4; i += PW * 32) {
          const long long t = t0 + (i & 3) * 32;
          if (t < T) {
            const long long n = t / F::S;
            prefetch_l2(F::pf_addr(a, n, (int)(t - n * F::S), i >> 2));
          }
        }
      }
      constexpr int ROWS = kBK / PW;
      float va[ROWS][4];
      auto gather = [&](int kb) {
#pragma unroll
        for (int q = 0; q < ROWS; ++q) {
          const int k = kb * kBK + warp * ROWS + q;
          const int kc = k < F::K ? k : F::K - 1;
          const typename F::BR R = F::Brow(a, kc);  // row context: once per (k-block, row)
#pragma unroll
          for (int mb = 0; mb < 4; ++mb) {
            const float v = F::Bk(a, R, (long long)pn[mb], ps[mb]);
            const bool ok = ((okmask >> mb) & 1u) && k < F::K;
            va[q][mb] = ok ? v : 0.f;
            // operand write-back for the wgrad (coalesced along the lane = pixel)
            if constexpr (F::SAVE_B) {
              if (ok) F::save_b(a, (long long)pn[mb], k, ps[mb], v);
            }
          }
        }
      };
      gather(0);
      for (int kb = 0; kb < KB; ++kb) {
        const int st = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
        uint8_t* sa_hi = smem + st * L::STAGE;
        uint8_t* sa_lo = sa_hi + L::A_BYTES;
#pragma unroll
        for (int q = 0; q < ROWS; ++q)
#pragma unroll
          for (int mb = 0; mb < 4; ++mb) {
            float h, l;
            split_tf32(va[q][mb], h, l);
            const int off = mn_off(mb * 32 + lane, warp * ROWS + q);
            *reinterpret_cast<float*>(sa_hi + off) = h;
            *reinterpret_cast<float*>(sa_lo + off) = l;
          }
        fence_async_smem();
        mbar_arrive(&full[st]);
        if (kb + 1 < KB) gather(kb + 1);
      }
    } else {
    const int r = p & (kBM - 1);        // tile row (pixel)
    const int half = p >> 7;            // 16 k of the 32-wide k-block
    const long long t = t0 + r;
    const bool ok = t < T;
    const long long n = ok ? t / F::S : 0;
    const int s = ok ? (int)(t - n * F::S) : 0;
    constexpr int WR = PACKED ? 0 : (NT + kBM - 1) / kBM;  // weight rows per thread (unpacked path)
    float va[16], vb[WR > 0 ? WR : 1][16];
    // Gather one k-block into registers: every address is clamped in range, the
    // value selected afterwards, so all loads issue back to back (no branches)
    // and overlap the wait for the ring slot.
    auto gather = [&](int kb) {
      const int kbase = kb * kBK + half * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = kbase + i;
        const float v = F::B(a, n, k < F::K ? k : F::K - 1, s);
        va[i] = (ok && k < F::K) ? v : 0.f;
      }
#pragma unroll
      for (int w = 0; w < WR; ++w) {
        const int row = r + w * kBM;
        const int col = c0 + row;
        const int cl = col < F::M ? col : F::M - 1;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int k = kbase + i;
          const float v = F::A(a, cl, k < F::K ? k : F::K - 1);
          vb[w][i] = (row < NT && col < F::M && k < F::K) ? v : 0.f;
        }
      }
    };
    gather(0);
    for (int kb = 0; kb < KB; ++kb) {
      const int st = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
      uint8_t* sa_hi = smem + st * L::STAGE;
      uint8_t* sa_lo = sa_hi + L::A_BYTES;
      uint8_t* sb_hi = sa_lo + L::A_BYTES;
      uint8_t* sb_lo = sb_hi + L::B_BYTES;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        float h[4], l[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) split_tf32(va[cc * 4 + j], h[j], l[j]);
        const int off = swz(r, half * 4 + cc);
        *reinterpret_cast<float4*>(sa_hi + off) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(sa_lo + off) = make_float4(l[0], l[1], l[2], l[3]);
      }
#pragma unroll
      for (int w = 0; w < WR; ++w) {
        const int row = r + w * kBM;
        if (row < NT) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            float h[4], l[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) split_tf32(vb[w][cc * 4 + j], h[j], l[j]);
            const int off = swz(row, half * 4 + cc);
            *reinterpret_cast<float4*>(sb_hi + off) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(sb_lo + off) = make_float4(l[0], l[1], l[2], l[3]);
          }
        }
      }
      fence_async_smem();
      mbar_arrive(&full[st]);
      if (kb + 1 < KB) gather(kb + 1);
    }
    }
    }
    // epilogue: TMEM lane quadrant = warp % 4, column half = warp / 4
    mbar_wait(done, 0);
    fence_after();
    const int q = warp & 3;
    const int tr = q * 32 + lane;  // accumulator row owned by this thread
    const long long te = t0 + tr;
    const long long en = te < T ? te / SX : 0;
    const int es = te < T ? (int)(te - en * SX) : 0;
    const bool eok = te < T && (SX == F::S || es < F::S);
    constexpr int HALF = ((NT + 16 * (PW / 4) - 1) / (16 * (PW / 4))) * 16;  // columns per warpgroup, multiple of 16
    const int cbeg = (warp >> 2) * HALF;
    for (int cc = cbeg; cc < cbeg + HALF && cc < NT; cc += 16) {
      float v[16];
      tmem_ld16(tmem + ((cv_u32)(q * 32) << 16) + cc, v);
#pragma unroll
      for (int c2 = 1; c2 < NACC; ++c2) {
        float u[16];
        tmem_ld16(tmem + c2 * NT + ((cv_u32)(q * 32) << 16) + cc, u);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += u[j];
      }
      if (eok) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int col = c0 + cc + j;
          if (cc + j < NT && col < F::M) F::store(a, en, col, es, v[j]);
        }
      }
    }
  } else if (warp == PW) {
    if (lane == 0) mma_loop<NT, STAGES, A_MN, NACC>(smem, full, empty, done, tmem, KB);
  } else if (PACKED && lane == 0) {
    // B operand: pre-split, pre-swizzled weight tile images (tc_pack_b), one
    // TMA bulk copy of {hi, lo} per k-block
    const uint8_t* img = reinterpret_cast<const uint8_t*>(F::packed(a)) + (long long)blockIdx.y * KB * 2 * L::B_BYTES;
    for (int kb = 0; kb < KB; ++kb) {
      const int st = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
      uint8_t* sb_hi = smem + st * L::STAGE + 2 * L::A_BYTES;
      mbar_arrive_tx(&full[st], 2 * L::B_BYTES);
      bulk_g2s(sb_hi, img + (long long)kb * 2 * L::B_BYTES, 2 * L::B_BYTES, &full[st]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == PW) {
    fence_after();
    tmem_free<NCOLS>(tmem);
  }
}

// ---------------------------------------------------------------------------
// FC forward with the computed operand staged in TENSOR memory (tcgen05.mma with
// A from TMEM).  The producer thread of TMEM lane r evaluates pixel t0 + r for 16
// consecutive k of the k-block (warp w: lane quadrant w % 4, k half w / 4): every
// gather is a 128 B coalesced warp load and the split operand goes to TMEM with
// tcgen05.st — no shared-memory stores and no 16 B-stride lane patterns, which is
// what bounds the shared-memory path's producers (L1/TEX).  Weights: packed
// K-major SW128 images by bulk copy, as in tc_gemm_pix.  TMEM: NACC x NT
// accumulator columns, then STAGES x {A_hi 32, A_lo 32} columns.
// ---------------------------------------------------------------------------
template <int V>
struct IntC {
  static constexpr int value = V;
};
// KS consecutive k of k-block kb (share hs) at this thread's pixel
template <class F, int KS>
__device__ __forceinline__ void tmema_gather(const CanvasArgs& a, const int kb, const int hs, const long long n, const int s, const bool ok, float* v) {
#pragma unroll
  for (int i = 0; i < KS; ++i) {
    const int k = kb * tc::kBK + hs * KS + i;
    const int kc = k < F::K ? k : F::K - 1;
    const float x = F::Bk(a, F::Brow(a, kc), n, s);
    v[i] = (ok && k < F::K) ? x : 0.f;
  }
}

template <class F, int NT, int STAGES, int NACC = 1, int PW = 8, bool UNROLL = false>
__device__ __forceinline__ void tc_gemm_pix_tmema(const CanvasArgs& a) {
  using namespace tc;
  static_assert(PW == 4 || PW == 8 || PW == 16, "4 lane quadrants x (1, 2 or 4) k shares");
  constexpr int KS = 32 / (PW / 4);  // k of the k-block per producer thread
  constexpr int B_BYTES = NT * 128;
  constexpr int ACOL = NACC * NT;  // first A column
  constexpr int NCOLS = TmemCols<ACOL + 64 * STAGES>::value;
  static_assert(ACOL + 64 * STAGES <= 512, "TMEM: accumulators + A stages exceed 512 columns");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem(smem_raw);
  cv_u64* full = (cv_u64*)(smem + STAGES * 2 * B_BYTES);
  cv_u64* empty = full + STAGES;
  cv_u64* done = empty + STAGES;
  cv_u32* tslot = (cv_u32*)(done + 1);
  const int warp = warp_index(), lane = threadIdx.x & 31;
  constexpr int KB = (F::K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], PW * 32 + 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == PW) tmem_alloc<NCOLS>(tslot);
  fence_before();
  __syncthreads();
  fence_after();
  const cv_u32 tmem = *tslot;

  const long long T = a.n * (long long)F::S;
  const long long t0 = (long long)blockIdx.x * kBM;
  const int c0 = blockIdx.y * NT;
  const int q = warp & 3;

  if (warp < PW) {
    const int half = warp >> 2;  // k share
    const long long t = t0 + q * 32 + lane;  // this thread's pixel (TMEM lane q*32 + lane)
    const bool ok = t < T;
    const long long n = ok ? t / F::S : 0;
    const int s = ok ? (int)(t - n * F::S) : 0;
    const cv_u32 lane_base = tmem + ((cv_u32)(q * 32) << 16);
    // HC >= 0: the k share is a compile-time constant and the k-block loop is fully
    // unrolled (UNROLL: the lowering's K <= TMEMA_UNROLL_MAX), so every k of the producer is a constant and
    // the functor's row context (channel / tap decomposition, plane offsets) folds
    // into immediates: per element only the gathers, the combine and the split remain
    auto produce = [&](auto hc) {
      constexpr int HC = decltype(hc)::value;
      constexpr int UF = HC >= 0 ? KB : 1;
      const int hs = HC >= 0 ? HC : half;
      float hi[KS], lo[KS], v[KS];
      tmema_gather<F, KS>(a, 0, hs, n, s, ok, v);
#pragma unroll UF
      for (int kb = 0; kb < KB; ++kb) {
        const int st = kb % STAGES;
#pragma unroll
        for (int i = 0; i < KS; ++i) split_tf32(v[i], hi[i], lo[i]);
        if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
        fence_after();
        const cv_u32 acol = lane_base + ACOL + st * 64 + hs * KS;
        if constexpr (KS >= 16) {
#pragma unroll
          for (int j = 0; j < KS; j += 16) {
            tmem_st16(acol + j, hi + j);
            tmem_st16(acol + 32 + j, lo + j);
          }
        } else {
          tmem_st8(acol, hi);
          tmem_st8(acol + 32, lo);
        }
        tmem_st_wait();
        fence_before();
        mbar_arrive(&full[st]);
        if (kb + 1 < KB) tmema_gather<F, KS>(a, kb + 1, hs, n, s, ok, v);
      }
    };
    if constexpr (UNROLL && PW == 8) {
      if (half == 0) produce(IntC<0>{});
      else produce(IntC<1>{});
    } else if constexpr (UNROLL && PW == 16) {
      if (half == 0) produce(IntC<0>{});
      else if (half == 1) produce(IntC<1>{});
      else if (half == 2) produce(IntC<2>{});
      else produce(IntC<3>{});
    } else {
      produce(IntC<-1>{});
    }
    // epilogue: TMEM lane quadrant = q, column half = warp / 4
    mbar_wait(done, 0);
    fence_after();
    const long long te = t0 + q * 32 + lane;
    const bool eok = te < T;
    const long long en = eok ? te / F::S : 0;
    const int es = eok ? (int)(te - en * F::S) : 0;
    constexpr int HALF = ((NT + 16 * (PW / 4) - 1) / (16 * (PW / 4))) * 16;
    const int cbeg = half * HALF;
    for (int cc = cbeg; cc < cbeg + HALF && cc < NT; cc += 16) {
      float r[16];
      tmem_ld16(tmem + ((cv_u32)(q * 32) << 16) + cc, r);
#pragma unroll
      for (int c2 = 1; c2 < NACC; ++c2) {
        float u[16];
        tmem_ld16(tmem + c2 * NT + ((cv_u32)(q * 32) << 16) + cc, u);
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] += u[j];
      }
      if (eok) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int col = c0 + cc + j;
          if (cc + j < NT && col < F::M) F::store(a, en, col, es, r[j]);
        }
      }
    }
  } else if (warp == PW) {
    if (lane == 0) {
      constexpr cv_u32 idesc = idesc_tf32(NT, false);
      for (int kb = 0; kb < KB; ++kb) {
        const int acc = (kb * NACC) / KB;
        const bool fresh = kb == 0 || ((kb - 1) * NACC) / KB != acc;
        const cv_u32 d = tmem + acc * NT;
        const int st = kb % STAGES;
        mbar_wait(&full[st], (kb / STAGES) & 1);
        fence_after();
        const cv_u32 a_hi = tmem + ACOL + st * 64;
        const cv_u32 b_hi = smem_u32(smem + st * 2 * B_BYTES);
        const cv_u32 b_lo = b_hi + B_BYTES;
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          mma_tf32_ts(d, a_hi + kk * 8, desc_k_sw128(b_hi + kk * 32), idesc, !(fresh && kk == 0));
          mma_tf32_ts(d, a_hi + kk * 8, desc_k_sw128(b_lo + kk * 32), idesc, 1);
          mma_tf32_ts(d, a_hi + 32 + kk * 8, desc_k_sw128(b_hi + kk * 32), idesc, 1);
        }
        commit(&empty[st]);
      }
      commit(done);
    }
  } else if (lane == 0) {
    // packed weight tile images, one bulk copy of {hi, lo} per k-block
    const uint8_t* img = reinterpret_cast<const uint8_t*>(F::packed(a)) + (long long)blockIdx.y * KB * 2 * B_BYTES;
    for (int kb = 0; kb < KB; ++kb) {
      const int st = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
      mbar_arrive_tx(&full[st], 2 * B_BYTES);
      bulk_g2s(smem + st * 2 * B_BYTES, img + (long long)kb * 2 * B_BYTES, 2 * B_BYTES, &full[st]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == PW) {
    fence_after();
    tmem_free<NCOLS>(tmem);
  }
}

// ---------------------------------------------------------------------------
// Persistent FC forward / dgrad (tcgen05, 3xTF32).  Same math and operand
// layouts as tc_gemm_pix<..., PACKED=true, A_MN=true>, but each CTA walks a
// strided list of (pixel tile, column tile) work items with two TMEM
// accumulators, so the epilogue of tile i (dedicated warps) overlaps the
// producer/MMA mainloop of tile i+1.  Warp roles: PW producer warps, 1 MMA
// warp, 1 TMA bulk-copy warp (packed weight images), 4 epilogue warps (one
// per TMEM lane quadrant).
// ---------------------------------------------------------------------------
template <int NT, int STAGES>
struct SmemP {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = NT * 128;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE;
  static constexpr int BYTES = BAR_OFF + (2 * STAGES + 16) * 8 + 16 + 1024;  // + up to 8 TMEM buffers' full/empty
};

template <class F, int NT, int STAGES, int PW, int EW>
__device__ __forceinline__ void tc_gemm_pix_persistent(const CanvasArgs& a) {
  using namespace tc;
  using L = SmemP<NT, STAGES>;
  // TMEM accumulators: 2 (double buffer), or EPI_NBUF for the broadcast-adjoint
  // epilogue, where EPI_WPB warpgroups share each buffer (column halves of a tile)
  constexpr int NB = F::EPI_BC ? F::EPI_NBUF : 2;
  static_assert(NB >= 2 && NB <= 8 && NB * NT <= 512, "TMEM buffers must fit 512 columns");
  constexpr int NCOLS = TmemCols<NB * NT>::value;
  constexpr int KB = (F::K + kBK - 1) / kBK;
  constexpr int NCT = (F::M + NT - 1) / NT;
  constexpr int ROWS = kBK / PW;  // k-rows per producer warp per k-block
  static_assert(kBK % PW == 0, "producer warps must divide the k-block");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem(smem_raw);
  cv_u64* full = (cv_u64*)(smem + L::BAR_OFF);
  cv_u64* empty = full + STAGES;
  cv_u64* tfull = empty + STAGES;   // [NB]
  cv_u64* tempty = tfull + 8;       // [NB]
  cv_u32* tslot = (cv_u32*)(tempty + 8);
  const int warp = warp_index(), lane = threadIdx.x & 31;
  const long long T = a.n * (long long)F::S;
  const long long PT = (T + kBM - 1) / kBM;
  const long long TILES = PT * NCT;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], PW * 32 + 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], (F::EPI_BC ? 4 * F::EPI_WPB : EW) * 32);  // EPI_BC: the buffer's warpgroups drain a tile
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == PW) tmem_alloc<NCOLS>(tslot);
  fence_before();
  __syncthreads();
  fence_after();
  const cv_u32 tmem = *tslot;

  if (warp < PW) {
   if constexpr (F::VEC) {
    // ---- producers, 4-pixel functor: lane owns tile pixels 4*lane .. 4*lane+3.
    // The CTA's (tile, k-block) work is one sequence g = 0 .. NG-1 (ring position g).
    const long long my_tiles = blockIdx.x < TILES ? (TILES - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long NG = my_tiles * KB;
    struct Pix {
      int kb, pn, ps;
      bool ok;
    };
    auto pix = [&](long long g) {
      Pix P;
      const long long tile = blockIdx.x + (g / KB) * gridDim.x;
      P.kb = (int)(g % KB);
      const long long tq = (tile / NCT) * kBM + 4 * lane;
      P.ok = tq < T;
      P.pn = P.ok ? (int)(tq / F::S) : 0;
      P.ps = P.ok ? (int)(tq - (long long)P.pn * F::S) : 0;
      return P;
    };
    auto row = [&](int kb, int q) {
      const int k = kb * kBK + warp * ROWS + q;
      return F::B4row(a, k < F::K ? k : F::K - 1);
    };
    auto put = [&](long long g, const Pix& P, float (&va)[ROWS][4]) {
      const int st = (int)(g % STAGES);
      if (g >= STAGES) mbar_wait(&empty[st], (cv_u32)(((g / STAGES) & 1) ^ 1));
      uint8_t* sa_hi = smem + st * L::STAGE;
      uint8_t* sa_lo = sa_hi + L::A_BYTES;
#pragma unroll
      for (int q = 0; q < ROWS; ++q) {
        const bool ok = P.ok && P.kb * kBK + warp * ROWS + q < F::K;
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_tf32(ok ? va[q][e] : 0.f, h[e], l[e]);
        const int off = mn_off(4 * lane, warp * ROWS + q);
        *reinterpret_cast<float4*>(sa_hi + off) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(sa_lo + off) = make_float4(l[0], l[1], l[2], l[3]);
      }
      fence_async_smem();
      mbar_arrive(&full[st]);
    };
    if constexpr (F::SPLIT) {
      constexpr int NB = F::B4NRAW;
      float x0[ROWS][NB], x1[ROWS][NB];
      Pix P0, P1;
      auto issue = [&](long long g, float (&x)[ROWS][NB], Pix& P) {
        P = pix(g);
#pragma unroll
        for (int q = 0; q < ROWS; ++q) F::B4ld(a, row(P.kb, q), (long long)P.pn, P.ps, x[q]);
      };
      auto commit_g = [&](long long g, const float (&x)[ROWS][NB], const Pix& P) {
        float va[ROWS][4];
#pragma unroll
        for (int q = 0; q < ROWS; ++q) F::B4cp(a, row(P.kb, q), x[q], va[q]);
        put(g, P, va);
      };
      if (NG > 0) issue(0, x0, P0);
      for (long long g = 0; g < NG; g += 2) {
        if (g + 1 < NG) issue(g + 1, x1, P1);
        commit_g(g, x0, P0);
        if (g + 1 < NG) {
          if (g + 2 < NG) issue(g + 2, x0, P0);
          commit_g(g + 1, x1, P1);
        }
      }
    } else {
      for (long long g = 0; g < NG; ++g) {
        const Pix P = pix(g);
        float va[ROWS][4];
#pragma unroll
        for (int q = 0; q < ROWS; ++q) F::B4k(a, row(P.kb, q), (long long)P.pn, P.ps, va[q]);
        put(g, P, va);
      }
    }
   } else {
    // ---- producers: MN-major computed operand, warp owns ROWS k-rows, lane = pixel
    long long g = 0;  // global k-block counter (ring position)
    for (long long tile = blockIdx.x; tile < TILES; tile += gridDim.x) {
      const long long t0 = (tile / NCT) * kBM;
      int pn[4], ps[4];
      unsigned okmask = 0;
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) {
        const long long t = t0 + mb * 32 + lane;
        okmask |= (t < T ? 1u : 0u) << mb;
        const long long tc = t < T ? t : T - 1;
        pn[mb] = (int)(tc / F::S);
        ps[mb] = (int)(tc - (long long)pn[mb] * F::S);
      }
      float va[ROWS][4];
      auto gather = [&](int kb) {
#pragma unroll
        for (int q = 0; q < ROWS; ++q) {
          const int k = kb * kBK + warp * ROWS + q;
          const int kc = k < F::K ? k : F::K - 1;
          const typename F::BR R = F::Brow(a, kc);
#pragma unroll
          for (int mb = 0; mb < 4; ++mb) {
            const float v = F::Bk(a, R, (long long)pn[mb], ps[mb]);
            va[q][mb] = (((okmask >> mb) & 1u) && k < F::K) ? v : 0.f;
          }
        }
      };
      gather(0);
      for (int kb = 0; kb < KB; ++kb, ++g) {
        const int st = (int)(g % STAGES);
        if (g >= STAGES) mbar_wait(&empty[st], (cv_u32)(((g / STAGES) & 1) ^ 1));
        uint8_t* sa_hi = smem + st * L::STAGE;
        uint8_t* sa_lo = sa_hi + L::A_BYTES;
#pragma unroll
        for (int q = 0; q < ROWS; ++q)
#pragma unroll
          for (int mb = 0; mb < 4; ++mb) {
            float h, l;
            split_tf32(va[q][mb], h, l);
            const int off = mn_off(mb * 32 + lane, warp * ROWS + q);
            *reinterpret_cast<float*>(sa_hi + off) = h;
            *reinterpret_cast<float*>(sa_lo + off) = l;
          }
        fence_async_smem();
        mbar_arrive(&full[st]);
        if (kb + 1 < KB) gather(kb + 1);
      }
    }
   }
  } else if (warp == PW) {
    // ---- MMA issuer
    if (lane == 0) {
      constexpr cv_u32 idesc = idesc_tf32(NT, true);
      long long g = 0;
      int it = 0;
      for (long long tile = blockIdx.x; tile < TILES; tile += gridDim.x, ++it) {
        const int buf = it % NB;
        if (it >= NB) mbar_wait(&tempty[buf], (cv_u32)(((it / NB) & 1) ^ 1));
        fence_after();
        const cv_u32 d = tmem + buf * NT;
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int st = (int)(g % STAGES);
          mbar_wait(&full[st], (cv_u32)((g / STAGES) & 1));
          fence_after();
          const cv_u32 a_hi = smem_u32(smem + st * L::STAGE);
          const cv_u32 a_lo = a_hi + L::A_BYTES;
          const cv_u32 b_hi = a_lo + L::A_BYTES;
          const cv_u32 b_lo = b_hi + L::B_BYTES;
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const cv_u64 dah = desc_mn_sw128_32b(a_hi + kk * 4096, 512, 2048);
            const cv_u64 dal = desc_mn_sw128_32b(a_lo + kk * 4096, 512, 2048);
            mma_tf32(d, dah, desc_k_sw128(b_hi + kk * 32), idesc, (kb | kk) != 0);
            mma_tf32(d, dah, desc_k_sw128(b_lo + kk * 32), idesc, 1);
            mma_tf32(d, dal, desc_k_sw128(b_hi + kk * 32), idesc, 1);
          }
          commit(&empty[st]);
        }
        commit(&tfull[buf]);
      }
    }
  } else if (warp == PW + 1) {
    // ---- TMA bulk loader of the packed weight tile images
    if (lane == 0) {
      const uint8_t* img0 = reinterpret_cast<const uint8_t*>(F::packed(a));
      long long g = 0;
      for (long long tile = blockIdx.x; tile < TILES; tile += gridDim.x) {
        const int ct = (int)(tile % NCT);
        const uint8_t* img = img0 + (long long)ct * KB * 2 * L::B_BYTES;
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int st = (int)(g % STAGES);
          if (g >= STAGES) mbar_wait(&empty[st], (cv_u32)(((g / STAGES) & 1) ^ 1));
          mbar_arrive_tx(&full[st], 2 * L::B_BYTES);
          bulk_g2s(smem + st * L::STAGE + 2 * L::A_BYTES, img + (long long)kb * 2 * L::B_BYTES, 2 * L::B_BYTES, &full[st]);
        }
      }
    }
  } else {
    // ---- epilogue: warp quadrant q = warp % 4 owns accumulator rows 32q..32q+31;
    // with EW = 8 the two warpgroups split the columns
    const int q = warp & 3;
    const int part = (warp - PW - 2) >> 2;  // 0 .. EW/4-1
    if constexpr (F::EPI_BC) {
      // broadcast-adjoint epilogue: TMEM columns of a tile are m*JT + jj (replica m
      // of lhs index j0 + jj), so the thread owning a pixel row writes the rhs
      // contribution of every column and sums the lhs terms over the replicas in
      // registers.  Warpgroups take alternate tiles (= alternate TMEM buffers).
      // warpgroup `part` drains buffer part / WPB (tiles it = buffer mod NB) and
      // its column share (lhs indices jj = (part % WPB) * JW .. + JW of each replica)
      constexpr int WPB = F::EPI_WPB, JW = F::EPI_JT / WPB, MR = F::EPI_M;
      constexpr int JT = JW;
      static_assert(EW == 4 * NB * WPB, "EPI_BC: EW = 4 x buffers x warpgroups per buffer");
      static_assert(JW == 8 || JW == 16, "column group of 8 or 16 per warpgroup");
      const int mybuf = part / WPB;
      int it = 0;
      for (long long tile = blockIdx.x; tile < TILES; tile += gridDim.x, ++it) {
        if (it % NB != mybuf) continue;
        const int buf = mybuf;
        const long long t0 = (tile / NCT) * kBM;
        const int j0 = (int)(tile % NCT) * F::EPI_JT + (part % WPB) * JW;
        const long long te = t0 + q * 32 + lane;
        const bool eok = te < T;
        const long long en = eok ? te / F::S : 0;
        const int es = eok ? (int)(te - en * F::S) : 0;
        // operand values do not depend on the GEMM: the lhs row and replica 0's rhs
        // gathers are issued before the accumulator is waited on, replica m+1's
        // while replica m is combined (two register sets, loop unrolled by 2).
        // Rows past the batch read a clamped pixel and only their stores are
        // predicated off, so the body stays branch-free.
        // per-pixel parts of the functors (image bases, pixel decomposition, lane
        // pointers), once per tile; the per-column rest runs on uniform registers
        const auto XL = F::epi_lhs_ctx(a, en, es);
        const auto XR = F::epi_rhs_ctx(a, en, es);
        const auto XT = F::epi_term_ctx(a, en, es);
        const auto XS = F::epi_store_l_ctx(a, en, es);
        float lv[JT], dl[JT], r0[JT], r1[JT];
#pragma unroll
        for (int jj = 0; jj < JT; ++jj) {
          lv[jj] = F::epi_lhs(a, XL, j0 + jj);
          r0[jj] = F::epi_rhs(a, XR, 0, j0 + jj);
          dl[jj] = 0.f;
        }
        mbar_wait(&tfull[buf], (cv_u32)((it / NB) & 1));
        fence_after();
        // ok: store predicate — the constant true on full tiles (no per-element branch)
        auto step = [&](int m, float (&rc)[JT], float (&rn)[JT], const bool ok) {
          if constexpr (F::EPI_PF) {
            const int mn = m + 1 < MR ? m + 1 : m;
#pragma unroll
            for (int jj = 0; jj < JT; ++jj) rn[jj] = F::epi_rhs(a, XR, mn, j0 + jj);
          } else if (m > 0) {
#pragma unroll
            for (int jj = 0; jj < JT; ++jj) rc[jj] = F::epi_rhs(a, XR, m, j0 + jj);
          }
          float g[JT];
          const cv_u32 ta = tmem + buf * NT + ((cv_u32)(q * 32) << 16) + m * F::EPI_JT + (part % WPB) * JW;
          if constexpr (JT == 16) tmem_ld16(ta, g);
          else tmem_ld8(ta, g);
#pragma unroll
          for (int jj = 0; jj < JT; ++jj) dl[jj] += F::epi_term(a, XT, m, j0 + jj, g[jj], lv[jj], rc[jj], ok);
        };
        if (t0 + kBM <= T) {
#pragma unroll 1
          for (int m = 0; m < MR; m += 2) {
            step(m, r0, r1, true);
            if (m + 1 < MR) step(m + 1, r1, r0, true);
          }
        } else {
#pragma unroll 1
          for (int m = 0; m < MR; m += 2) {
            step(m, r0, r1, eok);
            if (m + 1 < MR) step(m + 1, r1, r0, eok);
          }
        }
        fence_before();
        mbar_arrive(&tempty[buf]);
#pragma unroll
        for (int jj = 0; jj < JT; ++jj) F::epi_store_l(a, XS, j0 + jj, dl[jj], eok);
      }
    } else {
    constexpr int CPART = ((NT / (EW / 4)) + 31) / 32 * 32;
    int it = 0;
    for (long long tile = blockIdx.x; tile < TILES; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      const long long t0 = (tile / NCT) * kBM;
      const int c0 = (int)(tile % NCT) * NT;
      mbar_wait(&tfull[buf], (cv_u32)((it >> 1) & 1));
      fence_after();
      const long long te = t0 + q * 32 + lane;
      const bool eok = te < T;
      const long long en = eok ? te / F::S : 0;
      const int es = eok ? (int)(te - en * F::S) : 0;
      const int cb = part * CPART;
#pragma unroll 1
      for (int cc = cb; cc < cb + CPART && cc < NT; cc += 32) {
        float v[32];
        tmem_ld32(tmem + buf * NT + ((cv_u32)(q * 32) << 16) + cc, v);
        if (eok) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = c0 + cc + j;
            if (cc + j < NT && col < F::M) F::store(a, en, col, es, v[j]);
          }
        }
      }
      fence_before();
      mbar_arrive(&tempty[buf]);
    }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == PW) {
    fence_after();
    tmem_free<NCOLS>(tmem);
  }
}

// Pack the weight operand A(m,k) of a tc_gemm_pix launch into per-(column tile,
// k-block) images of the swizzled smem layout: [hi NT x 128 B][lo NT x 128 B],
// so the GEMM streams them with TMA bulk copies instead of per-row gathers.
template <class F, int NT>
__device__ __forceinline__ void tc_pack_b(const CanvasArgs& a) {
  constexpr int KB = (F::K + tc::kBK - 1) / tc::kBK;
  constexpr int NCT = (F::M + NT - 1) / NT;
  constexpr int BB = NT * 128;
  constexpr long long TOTAL = (long long)NCT * KB * NT * tc::kBK;
  float* img = F::packed(a);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < TOTAL; i += (long long)gridDim.x * blockDim.x) {
    const int kk = (int)(i % tc::kBK);
    const long long rest = i / tc::kBK;
    const int row = (int)(rest % NT);
    const long long tile = rest / NT;  // ct * KB + kb
    const int kb = (int)(tile % KB);
    const int ct = (int)(tile / KB);
    const int col = ct * NT + row;
    const int k = kb * tc::kBK + kk;
    const float v = (col < F::M && k < F::K) ? F::A(a, col, k) : 0.f;
    float hi, lo;
    tc::split_tf32(v, hi, lo);
    uint8_t* base = reinterpret_cast<uint8_t*>(img) + tile * 2 * BB;
    const int off = tc::swz(row, kk >> 2) + (kk & 3) * 4;
    *reinterpret_cast<float*>(base + off) = hi;
    *reinterpret_cast<float*>(base + BB + off) = lo;
  }
}

// ---------------------------------------------------------------------------
// FC wgrad on tensor cores: P[z][m][j] = sum_{t in chunk z} A(n,m,s) B(n,j,s).
// MMA rows = 128 input channels j (operand B), MMA cols = NT output channels
// m (operand A), reduction over a TCHUNK slice of pixels t; partials are
// summed in order by reduce_partials (deterministic).
// ---------------------------------------------------------------------------
// JG > 1: each CTA owns JG row tiles of 128 input channels (TMEM columns
// JG*NT), so the A operand (output-channel gradients, NT rows) is gathered once
// per JG tiles instead of once per tile.
template <class F, int NT, int STAGES, int PW = tc::kProducerWarps, int JG = 1>
__device__ __forceinline__ void tc_gemm_wgrad(const CanvasArgs& a) {
  using namespace tc;
  using L = SmemW<NT, JG, STAGES>;
  constexpr bool STACK = wgrad_stack<NT>();
  constexpr int NCOLS = TmemCols<NT * JG * (STACK ? 2 : 1)>::value;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem(smem_raw);
  cv_u64* full = (cv_u64*)(smem + L::BAR_OFF);
  cv_u64* empty = full + STAGES;
  cv_u64* done = empty + STAGES;
  cv_u32* tslot = (cv_u32*)(done + 1);
  const int warp = warp_index(), lane = threadIdx.x & 31;

  // producer row grouping (F::B4CLS): the operand rows are handed to producer
  // slots sorted by their shift class (the run-time 4 B offset of their quads),
  // so the 4 rows a warp produces per instruction share it and the select in B4cp
  // is warp-uniform.  Rows keep their smem position; only the producer changes.
  // F::B4KEY: rows sorted by their gather offset instead, so the 4 rows one warp
  // instruction produces read the same lines (on seed-7 #1: the 3 column taps of
  // one unfold row share one 16 B-chunk window; wavefronts per LDG drop)
  constexpr bool PERM = F::VEC && F::SPLIT && (F::B4CLS || F::B4KEY);
  __shared__ int perm_s[PERM ? kBM * JG : 1];
  __shared__ int cls_s[PERM ? kBM * JG : 1];
  if constexpr (PERM) {
    const int jbase = blockIdx.x * kBM * JG;
    for (int t = threadIdx.x; t < kBM * JG; t += blockDim.x) {
      const int jj = jbase + t;
      cls_s[t] = jj < F::J ? (F::B4CLS ? F::B4cls(F::B4row(a, jj)) : F::B4key(F::B4row(a, jj))) : 0x7fffffff;  // rows past J last
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kBM * JG; t += blockDim.x) {
      const int c = cls_s[t];
      int rank = 0;
      for (int u = 0; u < kBM * JG; ++u) {
        const int cu = cls_s[u];
        rank += (cu < c) || (cu == c && u < t);
      }
      perm_s[rank] = t;  // published by the barrier below
    }
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], PW * 32);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == PW) tmem_alloc<NCOLS>(tslot);
  fence_before();
  __syncthreads();
  fence_after();
  const cv_u32 tmem = *tslot;

  // F::SP: the vector producers enumerate (image, pixel) over a pixel range padded
  // to a multiple of 4 (pixels >= S are masked to zero by the functors)
  const bool vec_ok = F::VEC && (!F::NQ || (a.n & 3) == 0);
  const long long T = a.n * (long long)(vec_ok ? F::SP : F::S);
  const long long tbeg = (long long)blockIdx.z * F::TCHUNK;
  const long long tend = tbeg + F::TCHUNK < T ? tbeg + F::TCHUNK : T;
  const int KB = tend > tbeg ? (int)((tend - tbeg + kBK - 1) / kBK) : 0;
  const int j0 = blockIdx.x * kBM * JG;  // rows: input channels (JG tiles of 128)
  const int m0 = blockIdx.y * NT;        // cols: output channels

  // F::NQ: the functors' quads are 4 consecutive images at one pixel (S % 4 != 0);
  // the chunk's entries are then enumerated pixel-major (t = s * N + n) — the sum
  // over pixels does not care about the order — which needs N % 4 == 0, else the
  // scalar producers below run
  if constexpr (F::VEC) if (warp < PW && vec_ok) {
    // 4-pixel functors: lane = (row sub-index sub = lane / 8, pixel quad = lane % 8)
    // — a warp covers 4 rows x 32 pixels per pass, each thread one 16 B swizzle
    // chunk (4 consecutive pixels) of a row.  Row contexts are fixed for the CTA.
    constexpr int RP = PW * 4;  // rows per pass
    static_assert((kBM * JG) % RP == 0, "row passes must tile the 128-row MMA side");
    constexpr int RA = kBM * JG / RP, RB = (NT + RP - 1) / RP;
    const int quad = lane & 7, sub = lane >> 3;
    // operand-B row (smem row) of this thread's slot w
    int brow[RA];
#pragma unroll
    for (int w = 0; w < RA; ++w) {
      const int slot = warp * 4 + sub + RP * w;
      brow[w] = PERM ? perm_s[slot] : slot;
    }
    typename F::B4R rb[RA];
    typename F::A4R ra[RB];
#pragma unroll
    for (int w = 0; w < RA; ++w) {
      const int jj = j0 + brow[w];
      rb[w] = F::B4row(a, jj < F::J ? jj : F::J - 1);
    }
#pragma unroll
    for (int w = 0; w < RB; ++w) {
      const int mm = m0 + warp * 4 + sub + RP * w;
      ra[w] = F::A4row(a, mm < F::M ? mm : F::M - 1);
    }
    // split-precision stores of one k-block's operand quads into ring slot kb % STAGES
    auto put = [&](int kb, const float (&va)[RA][4], const float (&vb)[RB][4]) {
      const int st = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
      uint8_t* sa_hi = smem + st * L::STAGE;
      uint8_t* sa_lo = sa_hi + L::A_BYTES;
      uint8_t* sb_hi = sa_lo + L::A_BYTES;
      uint8_t* sb_lo = sb_hi + L::B_BYTES;
#pragma unroll
      for (int w = 0; w < RA; ++w) {
        const int row = brow[w];
        const int off = row * 128 + ((quad ^ (row & 7)) << 4);
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_tf32(va[w][e], h[e], l[e]);
        *reinterpret_cast<float4*>(sa_hi + off) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(sa_lo + off) = make_float4(l[0], l[1], l[2], l[3]);
      }
#pragma unroll
      for (int w = 0; w < RB; ++w) {
        const int row = warp * 4 + sub + RP * w;
        if (row < NT) {
          const int off = row * 128 + ((quad ^ (row & 7)) << 4);
          float h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) split_tf32(vb[w][e], h[e], l[e]);
          *reinterpret_cast<float4*>(sb_hi + off) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(sb_lo + off) = make_float4(l[0], l[1], l[2], l[3]);
        }
      }
      fence_async_smem();
      mbar_arrive(&full[st]);
    };
    // ok: the quad's valid lanes (bit e = pixel s + e); tend - tbeg is a multiple
    // of 4 (S or SP % 4 == 0, or N % 4 == 0 under NQ); padded pixels s + e >= S
    // feed zeros to the A side, so they add nothing to the sums
    auto pixel = [&](int kb, int& ok, int& n, int& s) {
      const long long t = tbeg + (long long)kb * kBK + 4 * quad;
      ok = t < tend ? 15 : 0;
      const int ti = (int)(ok ? t : tbeg);
      if constexpr (F::NQ) {
        s = ti / (int)a.n;
        n = ti - s * (int)a.n;
      } else {
        n = ti / F::SP;
        s = ti - n * F::SP;
        if constexpr (F::SP != F::S) ok &= (1 << (F::S - s < 4 ? F::S - s : 4)) - 1;
      }
    };
    if constexpr (F::SPLIT) {
      // software pipeline: the gathers of k-block kb+1 (raw registers, no use)
      // are issued before k-block kb is combined, split and stored
      constexpr int NB = F::B4NRAW, NA = F::A4NRAW;
      float xb0[RA][NB], xa0[RB][NA], xb1[RA][NB], xa1[RB][NA];
      int ok0 = 0, ok1 = 0;
      auto issue = [&](int kb, float (&xb)[RA][NB], float (&xa)[RB][NA], int& okv) {
        int n, s;
        pixel(kb, okv, n, s);
#pragma unroll
        for (int w = 0; w < RA; ++w) {
          // rows past J feed accumulator rows that are never stored: not gathered
          if (j0 + brow[w] < F::J) F::B4ld(a, rb[w], (long long)n, s, xb[w]);
        }
#pragma unroll
        for (int w = 0; w < RB; ++w) F::A4ld(a, ra[w], (long long)n, s, xa[w]);
      };
      auto commit_kb = [&](int kb, const float (&xb)[RA][NB], const float (&xa)[RB][NA], int okv) {
        float va[RA][4], vb[RB][4];
#pragma unroll
        for (int w = 0; w < RA; ++w) {
          if (j0 + brow[w] < F::J) {
            F::B4cp(a, rb[w], xb[w], va[w]);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) va[w][e] = 0.f;
          }
        }
#pragma unroll
        for (int w = 0; w < RB; ++w) {
          F::A4cp(a, ra[w], xa[w], vb[w]);
          const int keep = warp * 4 + sub + RP * w < NT ? okv : 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) vb[w][e] = (keep >> e) & 1 ? vb[w][e] : 0.f;
        }
        put(kb, va, vb);
      };
      if (KB > 0) issue(0, xb0, xa0, ok0);
      for (int kb = 0; kb < KB; kb += 2) {
        if (kb + 1 < KB) issue(kb + 1, xb1, xa1, ok1);
        commit_kb(kb, xb0, xa0, ok0);
        if (kb + 1 < KB) {
          if (kb + 2 < KB) issue(kb + 2, xb0, xa0, ok0);
          commit_kb(kb + 1, xb1, xa1, ok1);
        }
      }
    } else {
      float va[RA][4], vb[RB][4];
      auto gather = [&](int kb) {
        int ok;
        int n, s;
        pixel(kb, ok, n, s);
#pragma unroll
        for (int w = 0; w < RA; ++w) {
          if (j0 + brow[w] < F::J) {
            F::B4k(a, rb[w], (long long)n, s, va[w]);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) va[w][e] = 0.f;
          }
        }
#pragma unroll
        for (int w = 0; w < RB; ++w) {
          F::A4k(a, ra[w], (long long)n, s, vb[w]);
          const int keep = warp * 4 + sub + RP * w < NT ? ok : 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) vb[w][e] = (keep >> e) & 1 ? vb[w][e] : 0.f;
        }
      };
      if (KB > 0) gather(0);
      for (int kb = 0; kb < KB; ++kb) {
        put(kb, va, vb);
        if (kb + 1 < KB) gather(kb + 1);
      }
    }
  }
  if (warp < PW) {
    if (!vec_ok) {
    // lane = pixel of the 32-pixel k-block (coalesced gathers, one pixel
    // decomposition per k-block); warp w owns rows w, w+8, ... (channel index
    // math is warp-uniform); each warp writes whole 128 B swizzled rows.
    constexpr int RA = kBM * JG / PW, RB = (NT + PW - 1) / PW;
    // row contexts (channel decomposition, tap and base offsets of each row the
    // warp owns) are fixed for the CTA: built once here, so a gathered element
    // costs only its per-pixel part (F::Ak / F::Bk)
    typename F::BR rb[RA];
    typename F::AR ra[RB];
#pragma unroll
    for (int w = 0; w < RA; ++w) {
      const int jj = j0 + warp + PW * w;
      rb[w] = F::Brow(a, jj < F::J ? jj : F::J - 1);
    }
#pragma unroll
    for (int w = 0; w < RB; ++w) {
      const int mm = m0 + warp + PW * w;
      ra[w] = F::Arow(a, mm < F::M ? mm : F::M - 1);
    }
    float va[RA], vb[RB];
    auto gather = [&](int kb) {
      const long long t = tbeg + (long long)kb * kBK + lane;
      const bool ok = t < tend;
      const long long tc = ok ? t : tbeg;
      const long long n = tc / F::S;
      const int s = (int)(tc - n * F::S);
      // rows past J / M read a clamped valid row: their accumulator rows and
      // columns are never stored, so only pixels past the chunk end need zeros —
      // and zeroing one operand (A, the fewer rows) zeroes their products
#pragma unroll
      for (int w = 0; w < RA; ++w) va[w] = j0 + warp + PW * w < F::J ? F::Bk(a, rb[w], n, s) : 0.f;  // rows past J: never stored
#pragma unroll
      for (int w = 0; w < RB; ++w) {
        const float v = F::Ak(a, ra[w], n, s);
        vb[w] = (ok && warp + PW * w < NT) ? v : 0.f;
      }
    };
    const int off_l = ((lane >> 2) << 4) | ((lane & 3) << 2);  // chunk/word of this pixel before the swizzle
    // warm L2 with the source rows of k-block kb (one 128 B line per row):
    // issued kPfDist k-blocks before the gathers of that k-block
    constexpr int kPfDist = 3;
    auto prefetch = [&](int kb) {
      if constexpr (F::NPF > 0) {
        const long long t = tbeg + (long long)kb * kBK;
        if (kb < KB && t < tend) {
          const long long n = t / F::S;
          const int s = (int)(t - n * F::S);
          for (int i = threadIdx.x; i < F::NPF; i += PW * 32) prefetch_l2(F::pf_addr(a, n, s, i));
        }
      }
    };
    for (int d = 1; d <= kPfDist; ++d) prefetch(d);
    if (KB > 0) gather(0);
    for (int kb = 0; kb < KB; ++kb) {
      const int st = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) & 1) ^ 1);
      uint8_t* sa_hi = smem + st * L::STAGE;
      uint8_t* sa_lo = sa_hi + L::A_BYTES;
      uint8_t* sb_hi = sa_lo + L::A_BYTES;
      uint8_t* sb_lo = sb_hi + L::B_BYTES;
#pragma unroll
      for (int w = 0; w < RA; ++w) {
        const int row = warp + PW * w;  // tile row >> 7, row & 127 inside it (tiles are contiguous)
        const int off = row * 128 + (off_l ^ (((PW % 8 == 0 ? warp : row) & 7) << 4));
        float h, l;
        split_tf32(va[w], h, l);
        *reinterpret_cast<float*>(sa_hi + off) = h;
        *reinterpret_cast<float*>(sa_lo + off) = l;
      }
#pragma unroll
      for (int w = 0; w < RB; ++w) {
        const int row = warp + PW * w;
        if (row < NT) {
          const int off = row * 128 + (off_l ^ (((PW % 8 == 0 ? warp : row) & 7) << 4));
          float h, l;
          split_tf32(vb[w], h, l);
          *reinterpret_cast<float*>(sb_hi + off) = h;
          *reinterpret_cast<float*>(sb_lo + off) = l;
        }
      }
      fence_async_smem();
      mbar_arrive(&full[st]);
      prefetch(kb + 1 + kPfDist);
      if (kb + 1 < KB) gather(kb + 1);
    }
    }
    mbar_wait(done, 0);
    fence_after();
    const int q = warp & 3;
    float* P = F::partials(a) + (long long)blockIdx.z * F::M * F::J;
    // (tile, 16-column chunk) units over the PW/4 warpgroups; warp quadrant q reads TMEM lanes q*32..
    constexpr int CH = (NT + 15) / 16;
    for (int u = warp >> 2; u < JG * CH; u += PW / 4) {
      const int g = u / CH, cc = (u - g * CH) * 16;
      const int jj = j0 + g * kBM + q * 32 + lane;
      float v[16];
      tmem_ld16(tmem + ((cv_u32)(q * 32) << 16) + g * (STACK ? 2 * NT : NT) + cc, v);
      if constexpr (STACK) {
        float u[16];
        tmem_ld16(tmem + ((cv_u32)(q * 32) << 16) + g * 2 * NT + NT + cc, u);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += u[j];
      }
      if (jj < F::J) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int mm = m0 + cc + j;
          if (cc + j < NT && mm < F::M) P[(long long)mm * F::J + jj] = KB > 0 ? v[j] : 0.f;
        }
      }
    }
  } else if (warp == PW && lane == 0) {
    if (KB > 0) mma_loop_w<NT, JG, STAGES>(smem, full, empty, done, tmem, KB);
    else tc::mbar_arrive(done);
  }
  fence_before();
  __syncthreads();
  if (warp == PW) {
    fence_after();
    tmem_free<NCOLS>(tmem);
  }
}

}  // namespace canvas
