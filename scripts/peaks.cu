// Measured compute peaks of this B200 for the roofline denominators
// (VERDICT r1 "next" #2: "measure the tcgen05 kind::tf32 dense peak and the
// FP32-FFMA peak, burst and sustained, with a hand-written kernel").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/peaks scripts/peaks.cu -lcuda
//   build/peaks [--seconds 4] > profiles/r02_peaks.json
//
// * tcgen05 dense MMA: one CTA per SM, one elected thread issues back-to-back
//   tcgen05.mma.cta_group::1 M=128 N=256 K=8 (tf32) / K=16 (bf16) from
//   operands resident in shared memory (no loads), accumulating in TMEM, and
//   commits to an mbarrier every 64 MMAs so the issue queue never runs dry.
//   FLOPs = 2*M*N*K per MMA.  kind::f16 (bf16) is measured the same way as a
//   cross-check against MEASURED_PEAKS.json's cuBLAS bf16 number.
// * FP32 FFMA: 8 independent FMA chains per thread, 1024 threads per SM.
// * burst = best of 10 short launches (~10 ms); sustained = median launch of a
//   back-to-back run lasting --seconds (clocks settle under the power cap).
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

typedef unsigned int u32;
typedef unsigned long long u64;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ u64 desc_k_sw128(u32 saddr) {
  u64 d = 0;
  d |= (u64)((saddr >> 4) & 0x3FFF);
  d |= (u64)1 << 16;
  d |= (u64)(1024 >> 4) << 32;
  d |= (u64)1 << 46;
  d |= (u64)2 << 61;
  return d;
}

template <bool TF32>
__global__ void __launch_bounds__(128, 1) mma_peak(int iters, unsigned* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ u64 bar[2];
  __shared__ u32 tslot;
  const int warp = threadIdx.x >> 5;
  // operands: A 128 rows x 128 B, B 256 rows x 128 B (one k-block), filled with
  // pseudo-random values in (-1, 1) — real data toggles the datapath like a GEMM
  // does (zero operands draw far less power and never meet the power cap)
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) {
    u32 h = (u32)i * 2654435761u ^ (blockIdx.x * 40503u + 0x9e3779b9u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    const float f = ((h & 0xffffff) / 16777216.0f) * 2.f - 1.f;
    u32 bits = __float_as_uint(f);
    if (!TF32) {  // two bf16 values per 32-bit word
      const float f2 = (((h >> 8) & 0xffff) / 65536.0f) * 2.f - 1.f;
      bits = (__float_as_uint(f) >> 16) | (__float_as_uint(f2) & 0xffff0000u);
    }
    reinterpret_cast<u32*>(smem)[i] = bits;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = tslot;
  if (threadIdx.x == 0) {
    const u32 a = smem_u32(smem), b = a + 128 * 128;
    // kind::tf32: A/B format 2; kind::f16 (bf16): A/B format 1; D fp32; N = 256, M = 128
    const u32 idesc = (1u << 4) | ((TF32 ? 2u : 1u) << 7) | ((TF32 ? 2u : 1u) << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    auto wait = [&](int g) {
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar[g & 1])), "r"((u32)((g >> 1) & 1)) : "memory");
    };
    int g = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const u64 da = desc_k_sw128(a + kk * 32), db = desc_k_sw128(b + kk * 32);
        if (TF32)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(it | kk));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(it | kk));
      }
      if ((it & 15) == 15 || it == iters - 1) {
        // commit group g; wait for group g-1: one group always queued behind the running one
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[g & 1])) : "memory");
        if (g >= 1) wait(g - 1);
        ++g;
      }
    }
    wait(g - 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    u32 r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (r == 0xdeadbeef) sink[blockIdx.x] = r;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

__global__ void __launch_bounds__(1024) ffma_peak(int iters, float* sink) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float m = 0.999f, c = 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
      a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
    }
  }
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.f) sink[blockIdx.x] = s;
}

struct Stat {
  double burst, sustained;
  int sustained_launches;
};

template <class Launch>
Stat measure(Launch launch, double flops_per_launch, double seconds) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) launch();
  cudaDeviceSynchronize();
  double best = 0;
  for (int i = 0; i < 10; ++i) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::max(best, flops_per_launch / (ms * 1e-3));
  }
  std::vector<double> rates;
  std::vector<cudaEvent_t> ev(2 * 4096);
  for (auto& e : ev) cudaEventCreate(&e);
  double elapsed = 0;
  int n = 0;
  while (elapsed < seconds && n < 4096) {
    cudaEventRecord(ev[2 * n]);
    launch();
    cudaEventRecord(ev[2 * n + 1]);
    cudaEventSynchronize(ev[2 * n + 1]);
    float ms;
    cudaEventElapsedTime(&ms, ev[2 * n], ev[2 * n + 1]);
    rates.push_back(flops_per_launch / (ms * 1e-3));
    elapsed += ms * 1e-3;
    ++n;
  }
  std::sort(rates.begin(), rates.end());
  return {best, rates[rates.size() / 2], n};
}

int main(int argc, char** argv) {
  double seconds = 4.0;
  for (int i = 1; i < argc; ++i)
    if (!strcmp(argv[i], "--seconds") && i + 1 < argc) seconds = atof(argv[++i]);
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  unsigned* sink;
  cudaMalloc(&sink, 4096 * sizeof(float));
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(mma_peak<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_peak<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int it_tf32 = 4096, it_bf16 = 4096;
  auto tf32 = [&] { mma_peak<true><<<sms, 128, smem>>>(it_tf32, sink); };
  auto bf16 = [&] { mma_peak<false><<<sms, 128, smem>>>(it_bf16, sink); };
  const double f_tf32 = 2.0 * 128 * 256 * 8 * 4 * (double)it_tf32 * sms;
  const double f_bf16 = 2.0 * 128 * 256 * 16 * 4 * (double)it_bf16 * sms;
  const int it_ffma = 4096;
  auto ffma = [&] { ffma_peak<<<sms * 2, 1024>>>(it_ffma, (float*)sink); };
  const double f_ffma = 2.0 * 8 * 16 * (double)it_ffma * 1024 * sms * 2;
  Stat t = measure(tf32, f_tf32, seconds), b = measure(bf16, f_bf16, seconds), f = measure(ffma, f_ffma, seconds);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_max_mhz\": %d,\n", prop.name, sms, clk / 1000);
  printf(" \"tf32_tcgen05_tflops\": %.1f, \"tf32_tcgen05_tflops_sustained\": %.1f,\n", t.burst / 1e12, t.sustained / 1e12);
  printf(" \"bf16_tcgen05_tflops\": %.1f, \"bf16_tcgen05_tflops_sustained\": %.1f,\n", b.burst / 1e12, b.sustained / 1e12);
  printf(" \"fp32_ffma_tflops\": %.2f, \"fp32_ffma_tflops_sustained\": %.2f,\n", f.burst / 1e12, f.sustained / 1e12);
  printf(" \"how\": \"scripts/peaks.cu: tcgen05.mma cta_group::1 M128 N256 from smem-resident pseudo-random operands, 1 CTA/SM, commit every 64 MMAs; FFMA 8 chains x 1024 threads x 2 CTAs/SM; burst = best of 10 launches, sustained = median launch over %.0f s back to back\",\n", seconds);
  printf(" \"sustained_launches\": [%d, %d, %d]}\n", t.sustained_launches, b.sustained_launches, f.sustained_launches);
  return 0;
}
