// Post-pass kernels of a replaced conv: training-mode BatchNorm2d with the
// activation (ReLU) and the residual add of the enclosing block fused in.
//
// SPEC.md:658 specifies a BN post-pass for `build_module`; SURVEY App. A.10
// keeps the backbone's own BN after every replaced conv.  Both are the same
// operation on the replaced conv's output, [N, C, H, W] fp32 (App. A.0), and
// it is a pure HBM-bound pass: per channel c over M = N*H*W elements
//
//   forward   mean, var (biased) -> y = act((x - mean) * invstd * gamma + beta [+ r])
//   backward  g = dy * [y > 0]; Sg = sum g; Sgx = sum g * xhat
//             dx = gamma * invstd * (g - Sg / M - xhat * Sgx / M); dr = g
//
// which are torch.nn.functional.batch_norm (training) semantics, including
// the running-stat update (unbiased variance, momentum) and relu'(0) = 0
// (App. A.5, taken on the output like torch's threshold_backward).
//
// Layout of the work: channel c is split into P slices of whole images; one
// 256-thread CTA per (slice, channel), C*P ~ 8 CTAs per SM.  Inside a slice
// a CTA streams image planes with 16-byte loads when H*W % 4 == 0, and packs
// several small planes (7x7, 14x14) into one pass of the CTA so every thread
// stays busy.  Reductions are deterministic: per-thread fp32 sums of
// mean-shifted values (shift = x[0, c, 0, 0]), a fixed-order warp/CTA tree in
// fp64, per-slice partials in a workspace, and a fixed-order sum of the P
// partials by every consumer CTA.  No atomics: identical inputs give
// identical bits.
//
// Launches: forward = stats + apply, backward = reduce + apply (4 per BN).

#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#include <algorithm>

#include "canvas_post.h"

namespace {

constexpr int kBlock = 256;

struct Geo {
  int N, C, HW, P, V, U;  // V = vector width (4 or 1), U = HW / V units per plane
};

__host__ Geo make_geo(int N, int C, int HW, int P) {
  Geo g{N, C, HW, P, 1, HW};
  if (HW % 4 == 0) {
    g.V = 4;
    g.U = HW / 4;
  }
  return g;
}

// Calls f(offset_in_elements, vector_index_unused) for every V-wide unit of
// channel c in slice p, each unit exactly once per CTA, in a fixed
// thread -> unit mapping.
template <int V, class Fn>
__device__ __forceinline__ void for_units(const Geo& g, int c, int p, Fn&& f) {
  const int n0 = (int)((long long)p * g.N / g.P);
  const int n1 = (int)((long long)(p + 1) * g.N / g.P);
  const long long plane = (long long)g.C * g.HW;
  if (g.U >= kBlock) {
    for (int n = n0; n < n1; ++n) {
      const long long base = (long long)n * plane + (long long)c * g.HW;
      for (int u = threadIdx.x; u < g.U; u += kBlock) f(base + (long long)u * V);
    }
  } else {
    const int ipb = kBlock / g.U;
    const int u = threadIdx.x % g.U;
    const int j = threadIdx.x / g.U;
    if (j < ipb)
      for (int n = n0 + j; n < n1; n += ipb) f((long long)n * plane + (long long)c * g.HW + (long long)u * V);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order CTA sum of two values; result valid in thread 0
__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double sa[kBlock / 32], sb[kBlock / 32];
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sa[w] = a;
    sb[w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0.0;
    b = 0.0;
    for (int i = 0; i < kBlock / 32; ++i) {
      a += sa[i];
      b += sb[i];
    }
  }
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// ---------------------------------------------------------------- forward
template <int V>
__global__ void __launch_bounds__(kBlock) bn_stats(Geo g, const float* __restrict__ x, double2* __restrict__ part) {
  const int c = blockIdx.y, p = blockIdx.x;
  const float k = __ldg(x + (long long)c * g.HW);  // shift: first element of the channel
  float s1 = 0.f, s2 = 0.f;
  for_units<V>(g, c, p, [&](long long off) {
    if (V == 4) {
      const float4 v = ld4(x + off);
      const float a = v.x - k, b = v.y - k, d = v.z - k, e = v.w - k;
      s1 += (a + b) + (d + e);
      s2 = fmaf(a, a, fmaf(b, b, fmaf(d, d, fmaf(e, e, s2))));
    } else {
      const float a = __ldg(x + off) - k;
      s1 += a;
      s2 = fmaf(a, a, s2);
    }
  });
  double a = s1, b = s2;
  block_sum2(a, b);
  if (threadIdx.x == 0) part[c * g.P + p] = make_double2(a, b);
}

struct FwdArgs {
  const float* x;
  const float* r;  // residual (nullable)
  float* y;
  const float* gamma;
  const float* beta;
  float* running_mean;  // nullable
  float* running_var;   // nullable
  float* save_mean;
  float* save_invstd;
  const double2* part;
  float momentum, eps;
  int relu;
  uint8_t* mask;  // nullable: ReLU mask bytes (y > 0) for the backward
};

template <int V>
__global__ void __launch_bounds__(kBlock) bn_apply(Geo g, FwdArgs a) {
  const int c = blockIdx.y, p = blockIdx.x;
  __shared__ float sh[2];
  if (threadIdx.x == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < g.P; ++i) {
      const double2 q = a.part[c * g.P + i];
      s1 += q.x;
      s2 += q.y;
    }
    const double m = (double)g.N * g.HW;
    const double k = (double)__ldg(a.x + (long long)c * g.HW);
    const double d = s1 / m;
    double var = s2 / m - d * d;
    var = var > 0.0 ? var : 0.0;
    const double mean = k + d;
    const double invstd = 1.0 / sqrt(var + (double)a.eps);
    sh[0] = (float)mean;
    sh[1] = (float)invstd;
    if (p == 0) {
      a.save_mean[c] = (float)mean;
      a.save_invstd[c] = (float)invstd;
      if (a.running_mean) {
        const double mo = a.momentum;
        a.running_mean[c] = (float)((1.0 - mo) * a.running_mean[c] + mo * mean);
        a.running_var[c] = (float)((1.0 - mo) * a.running_var[c] + mo * var * m / (m > 1.0 ? m - 1.0 : 1.0));
      }
    }
  }
  __syncthreads();
  const float mean = sh[0];
  const float sc = sh[1] * __ldg(a.gamma + c);
  const float bt = __ldg(a.beta + c);
  const bool relu = a.relu != 0;
  const float* __restrict__ r = a.r;
  for_units<V>(g, c, p, [&](long long off) {
    if (V == 4) {
      const float4 v = ld4(a.x + off);
      float4 o = make_float4(fmaf(v.x - mean, sc, bt), fmaf(v.y - mean, sc, bt), fmaf(v.z - mean, sc, bt), fmaf(v.w - mean, sc, bt));
      if (r) {
        const float4 q = ld4(r + off);
        o.x += q.x;
        o.y += q.y;
        o.z += q.z;
        o.w += q.w;
      }
      if (relu) {
        o.x = fmaxf(o.x, 0.f);
        o.y = fmaxf(o.y, 0.f);
        o.z = fmaxf(o.z, 0.f);
        o.w = fmaxf(o.w, 0.f);
      }
      st4(a.y + off, o);
      if (a.mask) *reinterpret_cast<uchar4*>(a.mask + off) = make_uchar4(o.x > 0.f, o.y > 0.f, o.z > 0.f, o.w > 0.f);
    } else {
      float o = fmaf(__ldg(a.x + off) - mean, sc, bt);
      if (r) o += __ldg(r + off);
      if (relu) o = fmaxf(o, 0.f);
      a.y[off] = o;
      if (a.mask) a.mask[off] = o > 0.f;
    }
  });
}

// --------------------------------------------------------------- backward
struct BwdArgs {
  const float* x;
  const float* y;  // forward output (ReLU mask); nullable when !relu
  const float* dy;
  const float* gamma;
  const float* save_mean;
  const float* save_invstd;
  float* dx;
  float* dr;  // residual grad (nullable)
  float* dgamma;
  float* dbeta;
  double2* part;
  int relu;
  const uint8_t* mask;  // nullable: ReLU mask bytes written by the forward (read instead of y)
};

template <int V>
__global__ void __launch_bounds__(kBlock) bn_bwd_reduce(Geo g, BwdArgs a) {
  const int c = blockIdx.y, p = blockIdx.x;
  const float mean = __ldg(a.save_mean + c), inv = __ldg(a.save_invstd + c);
  const bool relu = a.relu != 0;
  float sg = 0.f, sgx = 0.f;
  for_units<V>(g, c, p, [&](long long off) {
    if (V == 4) {
      float4 d = ld4(a.dy + off);
      if (relu && a.mask) {
        const uchar4 m = __ldg(reinterpret_cast<const uchar4*>(a.mask + off));
        d.x = m.x ? d.x : 0.f;
        d.y = m.y ? d.y : 0.f;
        d.z = m.z ? d.z : 0.f;
        d.w = m.w ? d.w : 0.f;
      } else if (relu) {
        const float4 m = ld4(a.y + off);
        d.x = m.x > 0.f ? d.x : 0.f;
        d.y = m.y > 0.f ? d.y : 0.f;
        d.z = m.z > 0.f ? d.z : 0.f;
        d.w = m.w > 0.f ? d.w : 0.f;
      }
      const float4 v = ld4(a.x + off);
      sg += (d.x + d.y) + (d.z + d.w);
      sgx = fmaf(d.x, (v.x - mean) * inv, fmaf(d.y, (v.y - mean) * inv, fmaf(d.z, (v.z - mean) * inv, fmaf(d.w, (v.w - mean) * inv, sgx))));
    } else {
      float d = __ldg(a.dy + off);
      if (relu && !(a.mask ? __ldg(a.mask + off) != 0 : __ldg(a.y + off) > 0.f)) d = 0.f;
      sg += d;
      sgx = fmaf(d, (__ldg(a.x + off) - mean) * inv, sgx);
    }
  });
  double s = sg, t = sgx;
  block_sum2(s, t);
  if (threadIdx.x == 0) a.part[c * g.P + p] = make_double2(s, t);
}

template <int V>
__global__ void __launch_bounds__(kBlock) bn_bwd_apply(Geo g, BwdArgs a) {
  const int c = blockIdx.y, p = blockIdx.x;
  __shared__ float sh[2];
  if (threadIdx.x == 0) {
    double s = 0.0, t = 0.0;
    for (int i = 0; i < g.P; ++i) {
      const double2 q = a.part[c * g.P + i];
      s += q.x;
      t += q.y;
    }
    const double m = (double)g.N * g.HW;
    sh[0] = (float)(s / m);
    sh[1] = (float)(t / m);
    if (p == 0) {
      a.dbeta[c] = (float)s;
      a.dgamma[c] = (float)t;
    }
  }
  __syncthreads();
  const float mg = sh[0], mgx = sh[1];
  const float mean = __ldg(a.save_mean + c), inv = __ldg(a.save_invstd + c);
  const float k = inv * __ldg(a.gamma + c);
  const bool relu = a.relu != 0;
  float* __restrict__ dr = a.dr;
  for_units<V>(g, c, p, [&](long long off) {
    if (V == 4) {
      float4 d = ld4(a.dy + off);
      if (relu && a.mask) {
        const uchar4 m = __ldg(reinterpret_cast<const uchar4*>(a.mask + off));
        d.x = m.x ? d.x : 0.f;
        d.y = m.y ? d.y : 0.f;
        d.z = m.z ? d.z : 0.f;
        d.w = m.w ? d.w : 0.f;
      } else if (relu) {
        const float4 m = ld4(a.y + off);
        d.x = m.x > 0.f ? d.x : 0.f;
        d.y = m.y > 0.f ? d.y : 0.f;
        d.z = m.z > 0.f ? d.z : 0.f;
        d.w = m.w > 0.f ? d.w : 0.f;
      }
      const float4 v = ld4(a.x + off);
      float4 o;
      o.x = k * (d.x - mg - (v.x - mean) * inv * mgx);
      o.y = k * (d.y - mg - (v.y - mean) * inv * mgx);
      o.z = k * (d.z - mg - (v.z - mean) * inv * mgx);
      o.w = k * (d.w - mg - (v.w - mean) * inv * mgx);
      st4(a.dx + off, o);
      if (dr) st4(dr + off, d);
    } else {
      float d = __ldg(a.dy + off);
      if (relu && !(a.mask ? __ldg(a.mask + off) != 0 : __ldg(a.y + off) > 0.f)) d = 0.f;
      a.dx[off] = k * (d - mg - (__ldg(a.x + off) - mean) * inv * mgx);
      if (dr) dr[off] = d;
    }
  });
}


// ------------------------------------------------------------- max-pool
// The stem max-pool of the ResNet backbones (3x3, stride 2, pad 1) between the
// fused stem BN+ReLU and the first replaced conv.  Forward: one thread per
// output, first maximum in row-major window order wins (NaN propagates, torch
// semantics), the winner's window slot kept as one byte.  Backward is a
// gather — each input element sums, in a fixed order, the gradients of the
// (at most ceil(K/S)^2) windows whose recorded winner it is: no atomics.
struct PoolGeo {
  int N, C, H, W, K, S, P, OH, OW;
};

// Plane-major grid (blockIdx.y strides over N*C planes, 32-bit index math in a
// plane); the common 3x3 / stride 2 / pad 1 stem is a compile-time instance
// (KK = 0: runtime geometry).
template <int KK, int SS, int PP>
__global__ void __launch_bounds__(kBlock) maxpool_fwd(PoolGeo g, const float* __restrict__ x, float* __restrict__ y,
                                                      uint8_t* __restrict__ idx) {
  const int K = KK ? KK : g.K, S = KK ? SS : g.S, P = KK ? PP : g.P;
  const int j = blockIdx.x * kBlock + threadIdx.x;
  if (j >= g.OH * g.OW) return;
  const int oh = j / g.OW, ow = j - oh * g.OW;
  const long long planes = (long long)g.N * g.C;
  for (long long pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const float* xp = x + pl * g.H * g.W;
    float m = -INFINITY;
    int best = 0;
#pragma unroll
    for (int kh = 0; kh < (KK ? KK : 15); ++kh) {
      if (!KK && kh >= K) break;
      const int h = oh * S - P + kh;
      if ((unsigned)h >= (unsigned)g.H) continue;
#pragma unroll
      for (int kw = 0; kw < (KK ? KK : 15); ++kw) {
        if (!KK && kw >= K) break;
        const int w = ow * S - P + kw;
        if ((unsigned)w >= (unsigned)g.W) continue;
        const float v = __ldg(xp + h * g.W + w);
        if (v > m || isnan(v)) {
          m = v;
          best = kh * K + kw;
        }
      }
    }
    const long long o = pl * g.OH * g.OW + j;
    y[o] = m;
    idx[o] = (uint8_t)best;
  }
}

// 3x3 / stride 2 / pad 1 backward in closed form: an even input row is covered
// by one window row (kh = 1), an odd one by two (kh = 2 then kh = 0), same for
// columns, so each input sums at most four window gradients (increasing oh, ow).
__global__ void __launch_bounds__(kBlock) maxpool_bwd_k3s2(PoolGeo g, const float* __restrict__ dy,
                                                          const uint8_t* __restrict__ idx, float* __restrict__ dx) {
  const int j = blockIdx.x * kBlock + threadIdx.x;
  if (j >= g.H * g.W) return;
  const int h = j / g.W, w = j - h * g.W;
  int rows = 1, oh0, kh0, oh1 = 0, kh1 = 0;
  if (h & 1) {
    oh0 = h >> 1, kh0 = 2, oh1 = (h + 1) >> 1, kh1 = 0;
    rows = oh1 < g.OH ? 2 : 1;
  } else {
    oh0 = h >> 1, kh0 = 1;
  }
  int cols = 1, ow0, kw0, ow1 = 0, kw1 = 0;
  if (w & 1) {
    ow0 = w >> 1, kw0 = 2, ow1 = (w + 1) >> 1, kw1 = 0;
    cols = ow1 < g.OW ? 2 : 1;
  } else {
    ow0 = w >> 1, kw0 = 1;
  }
  const long long planes = (long long)g.N * g.C;
  for (long long pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const float* dyp = dy + pl * g.OH * g.OW;
    const uint8_t* ip = idx + pl * g.OH * g.OW;
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r >= rows) break;
      const int oh = r ? oh1 : oh0, kh = r ? kh1 : kh0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c >= cols) break;
        const int o = oh * g.OW + (c ? ow1 : ow0);
        const int slot = kh * 3 + (c ? kw1 : kw0);
        const float d = __ldg(dyp + o);
        acc += __ldg(ip + o) == slot ? d : 0.f;
      }
    }
    dx[pl * g.H * g.W + j] = acc;
  }
}

// 3x3 / stride 2 / pad 1 forward, W % 4 == 0: two outputs per thread from one
// aligned float4 (input cols 4b..4b+3) + one scalar (col 4b-1) per window row;
// float2 / 2-byte stores.  Same scan order and NaN rule as maxpool_fwd.
__global__ void __launch_bounds__(kBlock) maxpool_fwd_k3s2_x2(PoolGeo g, const float* __restrict__ x, float* __restrict__ y,
                                                             uint8_t* __restrict__ idx) {
  const int OW2 = g.OW >> 1;
  const int j = blockIdx.x * kBlock + threadIdx.x;
  if (j >= g.OH * OW2) return;
  const int oh = j / OW2, b = j - oh * OW2;
  const long long planes = (long long)g.N * g.C;
#pragma unroll 2
  for (long long pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const float* xp = x + pl * g.H * g.W;
    float m0 = -INFINITY, m1 = -INFINITY;
    int b0 = 0, b1 = 0;
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int h = oh * 2 - 1 + kh;
      if ((unsigned)h >= (unsigned)g.H) continue;
      const float* row = xp + h * g.W + 4 * b;
      const float4 q = __ldg(reinterpret_cast<const float4*>(row));
      const float v[5] = {b > 0 ? __ldg(row - 1) : 0.f, q.x, q.y, q.z, q.w};
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        if (b > 0 || kw > 0) {  // output 2b: input col 4b-1+kw
          const float t = v[kw];
          if (t > m0 || isnan(t)) m0 = t, b0 = kh * 3 + kw;
        }
        const float t = v[kw + 2];  // output 2b+1: input col 4b+1+kw (< W: W % 4 == 0)
        if (t > m1 || isnan(t)) m1 = t, b1 = kh * 3 + kw;
      }
    }
    const long long o = pl * g.OH * g.OW + (long long)oh * g.OW + 2 * b;
    *reinterpret_cast<float2*>(y + o) = make_float2(m0, m1);
    *reinterpret_cast<uchar2*>(idx + o) = make_uchar2((uint8_t)b0, (uint8_t)b1);
  }
}

// 3x3 / stride 2 / pad 1 backward, W % 4 == 0: four consecutive inputs per thread
// (cols 4a'..4a'+3 read window cols a, a+1, a+2 with a = 2a'), float4 store.  Per
// element the window gradients are summed in the order of maxpool_bwd_k3s2.
__global__ void __launch_bounds__(kBlock) maxpool_bwd_k3s2_x4(PoolGeo g, const float* __restrict__ dy,
                                                             const uint8_t* __restrict__ idx, float* __restrict__ dx) {
  const int W4 = g.W >> 2;
  const int j = blockIdx.x * kBlock + threadIdx.x;
  if (j >= g.H * W4) return;
  const int h = j / W4, w0 = (j - h * W4) * 4;
  int rows = 1, oh0, kh0, oh1 = 0, kh1 = 0;
  if (h & 1) {
    oh0 = h >> 1, kh0 = 2, oh1 = (h + 1) >> 1, kh1 = 0;
    rows = oh1 < g.OH ? 2 : 1;
  } else {
    oh0 = h >> 1, kh0 = 1;
  }
  const int a = w0 >> 1;
  const bool c2 = a + 2 < g.OW;
  const long long planes = (long long)g.N * g.C;
#pragma unroll 2
  for (long long pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const float* dyp = dy + pl * g.OH * g.OW;
    const uint8_t* ip = idx + pl * g.OH * g.OW;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r >= rows) break;
      const int o = (r ? oh1 : oh0) * g.OW + a, k3 = (r ? kh1 : kh0) * 3;
      const float d0 = __ldg(dyp + o), d1 = __ldg(dyp + o + 1), d2 = c2 ? __ldg(dyp + o + 2) : 0.f;
      const int i0 = __ldg(ip + o), i1 = __ldg(ip + o + 1), i2 = c2 ? __ldg(ip + o + 2) : 255;
      acc.x += i0 == k3 + 1 ? d0 : 0.f;
      acc.y += i0 == k3 + 2 ? d0 : 0.f;
      acc.y += i1 == k3 ? d1 : 0.f;
      acc.z += i1 == k3 + 1 ? d1 : 0.f;
      acc.w += i1 == k3 + 2 ? d1 : 0.f;
      acc.w += i2 == k3 ? d2 : 0.f;
    }
    *reinterpret_cast<float4*>(dx + pl * g.H * g.W + h * g.W + w0) = acc;
  }
}

template <int KK, int SS, int PP>
__global__ void __launch_bounds__(kBlock) maxpool_bwd(PoolGeo g, const float* __restrict__ dy,
                                                      const uint8_t* __restrict__ idx, float* __restrict__ dx) {
  const int K = KK ? KK : g.K, S = KK ? SS : g.S, P = KK ? PP : g.P;
  const int j = blockIdx.x * kBlock + threadIdx.x;
  if (j >= g.H * g.W) return;
  const int h = j / g.W, w = j - h * g.W;
  const long long planes = (long long)g.N * g.C;
  for (long long pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const float* dyp = dy + pl * g.OH * g.OW;
    const uint8_t* ip = idx + pl * g.OH * g.OW;
    float acc = 0.f;
#pragma unroll
    for (int kh = (KK ? KK : 15) - 1; kh >= 0; --kh) {  // windows in increasing oh
      if (!KK && kh >= K) continue;
      const int t = h + P - kh;
      if (t < 0 || t % S) continue;
      const int oh = t / S;
      if (oh >= g.OH) continue;
#pragma unroll
      for (int kw = (KK ? KK : 15) - 1; kw >= 0; --kw) {
        if (!KK && kw >= K) continue;
        const int u = w + P - kw;
        if (u < 0 || u % S) continue;
        const int ow = u / S;
        if (ow >= g.OW) continue;
        const int o = oh * g.OW + ow;
        if (__ldg(ip + o) == kh * K + kw) acc += __ldg(dyp + o);
      }
    }
    dx[pl * g.H * g.W + j] = acc;
  }
}

thread_local char g_err[256];

int fail(const char* what, cudaError_t e) {
  snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
  return CANVAS_POST_ERR_CUDA;
}

int slices(int N, int C) {
  // ~8 CTAs per SM (148 SMs), whole images per slice
  int p = (148 * 8 + C - 1) / C;
  if (p > N) p = N;
  if (p < 1) p = 1;
  return p;
}

bool aligned16(const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

}  // namespace

extern "C" {

int canvas_post_abi_version(void) { return CANVAS_POST_ABI_VERSION; }

const char* canvas_post_last_error(void) { return g_err; }

size_t canvas_bn_workspace(int64_t N, int64_t C, int64_t HW) {
  (void)HW;
  return (size_t)slices((int)N, (int)C) * (size_t)C * sizeof(double2);
}

int canvas_bn_forward(int64_t N, int64_t C, int64_t HW, const float* x, const float* residual, float* y,
                      const float* gamma, const float* beta, float* running_mean, float* running_var,
                      float* save_mean, float* save_invstd, float momentum, float eps, int relu, uint8_t* relu_mask,
                      void* workspace, void* stream) {
  if (N < 1 || C < 1 || HW < 1 || !x || !y || !gamma || !beta || !save_mean || !save_invstd || !workspace ||
      (running_mean == nullptr) != (running_var == nullptr) || N * C * HW >= (1LL << 40)) {
    snprintf(g_err, sizeof g_err, "canvas_bn_forward: bad arguments");
    return CANVAS_POST_ERR_ARGS;
  }
  Geo g = make_geo((int)N, (int)C, (int)HW, slices((int)N, (int)C));
  if (!aligned16(x) || !aligned16(residual) || !aligned16(y)) g.V = 1, g.U = g.HW;
  cudaStream_t s = (cudaStream_t)stream;
  FwdArgs a{x, residual, y, gamma, beta, running_mean, running_var, save_mean, save_invstd, (const double2*)workspace, momentum, eps, relu, relu ? relu_mask : nullptr};
  const dim3 grid(g.P, g.C);
  if (g.V == 4) {
    bn_stats<4><<<grid, kBlock, 0, s>>>(g, x, (double2*)workspace);
    bn_apply<4><<<grid, kBlock, 0, s>>>(g, a);
  } else {
    bn_stats<1><<<grid, kBlock, 0, s>>>(g, x, (double2*)workspace);
    bn_apply<1><<<grid, kBlock, 0, s>>>(g, a);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CANVAS_POST_OK : fail("canvas_bn_forward launch", e);
}

int canvas_bn_backward(int64_t N, int64_t C, int64_t HW, const float* x, const float* y, const uint8_t* relu_mask,
                       const float* dy, const float* gamma, const float* save_mean, const float* save_invstd,
                       float* dx, float* dresidual, float* dgamma, float* dbeta, int relu, void* workspace,
                       void* stream) {
  if (N < 1 || C < 1 || HW < 1 || !x || !dy || !gamma || !save_mean || !save_invstd || !dx || !dgamma || !dbeta ||
      !workspace || (relu && !y && !relu_mask) || N * C * HW >= (1LL << 40)) {
    snprintf(g_err, sizeof g_err, "canvas_bn_backward: bad arguments");
    return CANVAS_POST_ERR_ARGS;
  }
  Geo g = make_geo((int)N, (int)C, (int)HW, slices((int)N, (int)C));
  if (!aligned16(x) || !aligned16(y) || !aligned16(dy) || !aligned16(dx) || !aligned16(dresidual)) g.V = 1, g.U = g.HW;
  cudaStream_t s = (cudaStream_t)stream;
  BwdArgs a{x, y, dy, gamma, save_mean, save_invstd, dx, dresidual, dgamma, dbeta, (double2*)workspace, relu, relu_mask};
  const dim3 grid(g.P, g.C);
  if (g.V == 4) {
    bn_bwd_reduce<4><<<grid, kBlock, 0, s>>>(g, a);
    bn_bwd_apply<4><<<grid, kBlock, 0, s>>>(g, a);
  } else {
    bn_bwd_reduce<1><<<grid, kBlock, 0, s>>>(g, a);
    bn_bwd_apply<1><<<grid, kBlock, 0, s>>>(g, a);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CANVAS_POST_OK : fail("canvas_bn_backward launch", e);
}

int canvas_maxpool2d_forward(int64_t N, int64_t C, int64_t H, int64_t W, int K, int S, int P, const float* x, float* y,
                             uint8_t* argmax, void* stream) {
  if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || K > 15 || S < 1 || P < 0 || 2 * P > K || !x || !y || !argmax) {
    snprintf(g_err, sizeof g_err, "canvas_maxpool2d_forward: bad arguments");
    return CANVAS_POST_ERR_ARGS;
  }
  PoolGeo g{(int)N, (int)C, (int)H, (int)W, K, S, P, (int)((H + 2 * P - K) / S + 1), (int)((W + 2 * P - K) / S + 1)};
  if (K == 3 && S == 2 && P == 1 && W % 4 == 0 && aligned16(x) && ((uintptr_t)y & 7u) == 0 && ((uintptr_t)argmax & 1u) == 0) {
    const int bx = (g.OH * (g.OW >> 1) + kBlock - 1) / kBlock;
    const dim3 grid(bx, (unsigned)std::min<long long>(N * C, std::max(1, 148 * 32 / bx)));
    maxpool_fwd_k3s2_x2<<<grid, kBlock, 0, (cudaStream_t)stream>>>(g, x, y, argmax);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CANVAS_POST_OK : fail("canvas_maxpool2d_forward launch", e);
  }
  const int bx = (g.OH * g.OW + kBlock - 1) / kBlock;
  const dim3 grid(bx, (unsigned)std::min<long long>(N * C, std::max(1, 148 * 32 / bx)));
  if (K == 3 && S == 2 && P == 1)
    maxpool_fwd<3, 2, 1><<<grid, kBlock, 0, (cudaStream_t)stream>>>(g, x, y, argmax);
  else
    maxpool_fwd<0, 0, 0><<<grid, kBlock, 0, (cudaStream_t)stream>>>(g, x, y, argmax);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CANVAS_POST_OK : fail("canvas_maxpool2d_forward launch", e);
}

int canvas_maxpool2d_backward(int64_t N, int64_t C, int64_t H, int64_t W, int K, int S, int P, const float* dy,
                              const uint8_t* argmax, float* dx, void* stream) {
  if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || K > 15 || S < 1 || P < 0 || 2 * P > K || !dy || !argmax || !dx) {
    snprintf(g_err, sizeof g_err, "canvas_maxpool2d_backward: bad arguments");
    return CANVAS_POST_ERR_ARGS;
  }
  PoolGeo g{(int)N, (int)C, (int)H, (int)W, K, S, P, (int)((H + 2 * P - K) / S + 1), (int)((W + 2 * P - K) / S + 1)};
  if (K == 3 && S == 2 && P == 1 && W % 4 == 0 && aligned16(dx)) {
    const int bx = (int)((H * (W >> 2) + kBlock - 1) / kBlock);
    const dim3 grid(bx, (unsigned)std::min<long long>(N * C, std::max(1, 148 * 32 / bx)));
    maxpool_bwd_k3s2_x4<<<grid, kBlock, 0, (cudaStream_t)stream>>>(g, dy, argmax, dx);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CANVAS_POST_OK : fail("canvas_maxpool2d_backward launch", e);
  }
  const int bx = (int)((H * W + kBlock - 1) / kBlock);
  const dim3 grid(bx, (unsigned)std::min<long long>(N * C, std::max(1, 148 * 32 / bx)));
  if (K == 3 && S == 2 && P == 1)
    maxpool_bwd_k3s2<<<grid, kBlock, 0, (cudaStream_t)stream>>>(g, dy, argmax, dx);
  else
    maxpool_bwd<0, 0, 0><<<grid, kBlock, 0, (cudaStream_t)stream>>>(g, dy, argmax, dx);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CANVAS_POST_OK : fail("canvas_maxpool2d_backward launch", e);
}

}  // extern "C"
