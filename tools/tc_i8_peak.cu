// int8 tcgen05 MMA throughput microbenchmark (development tool): one CTA per
// SM issues back-to-back tcgen05.mma.cta_group::1.kind::i8 (M = 128, K = 32,
// N = 64 / 128 / 256) from resident SWIZZLE_64B smem tiles into TMEM, no
// loads, no epilogue. Reports dense int8 TOP/s, i.e. the tensor roofline of
// the split conversion product (l2c_ozaki.cu) for each tile width.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --expt-relaxed-constexpr -o tools/tc_i8_peak tools/tc_i8_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (32ull << 32) | (1ull << 46) |
         (4ull << 61);
}

template <int N>
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  // A: 8 tiles of 128 x 64 B, B: 8 tiles of N x 64 B (zeros)
  const int bytes = 8 * (128 * 64) + 8 * (N * 64);
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  constexpr int NACC = 512 / N;  // accumulators that fit
  unsigned long long t0 = clock64();
  if (warp == 0) {
    const uint64_t ad0 = desc64(smem_u32(smem)), bd0 = desc64(smem_u32(smem + 8 * 128 * 64));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int m = 0; m < 72; ++m) {
        const int i = m % 8, j = (m / 8) % 8, ks = m & 1;
        const uint64_t ad = ad0 + (uint64_t)((i * 128 * 64 + ks * 32) >> 4);
        const uint64_t bd = bd0 + (uint64_t)((j * N * 64 + ks * 32) >> 4);
        const uint32_t d = tmem + (uint32_t)((m % NACC) * N);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
              smem_u32(&bar)));
      // wait for this batch (keeps <= 72 MMAs in flight, like one pipeline stage)
      asm volatile(
          "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(
              smem_u32(&bar)), "r"((uint32_t)(it & 1)));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// TS form (A from TMEM, as oz_gemm2_kernel): A tiles copied once into 8
// 8-column slots after 7 x N accumulator columns, then back-to-back MMAs.
template <int N, bool CP>
__global__ void __launch_bounds__(128, 1) peak_ts_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int bytes = 8 * (128 * 64) + 8 * (N * 64);
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  constexpr int NACC = 7;
  unsigned long long t0 = clock64();
  if (warp == 0) {
    const uint64_t ad0 = desc64(smem_u32(smem)), bd0 = desc64(smem_u32(smem + 8 * 128 * 64));
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(tmem + (uint32_t)(NACC * N + 8 * i)),
          "l"(ad0 + (uint64_t)((i * 128 * 64) >> 4)));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int m = 0; m < 72; ++m) {
        const int i = m % 8, j = (m / 8) % 8, ks = m & 1;
        const uint64_t bd = bd0 + (uint64_t)((j * N * 64 + ks * 32) >> 4);
        const uint32_t d = tmem + (uint32_t)((m % NACC) * N);
        const uint32_t a = tmem + (uint32_t)(NACC * N + 8 * i);
        if (CP && (m & 3) == 0)  // one A-tile copy per 4 MMAs (oz_gemm2: 7 per 28)
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(tmem + (uint32_t)(NACC * N + 8 * ((i + 4) & 7))),
              "l"(ad0 + (uint64_t)((((i + 4) & 7) * 128 * 64) >> 4)));
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(a), "l"(bd), "r"(idesc), "r"(1u));
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
              smem_u32(&bar)));
      asm volatile(
          "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(
              smem_u32(&bar)), "r"((uint32_t)(it & 1)));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, bool CP>
void run_ts(int sms) {
  const int smem = 8 * 128 * 64 + 8 * N * 64 + 1024;
  cudaFuncSetAttribute(peak_ts_kernel<N, CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  const int iters = 2000;
  peak_ts_kernel<N, CP><<<sms, 128, smem>>>(10, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  peak_ts_kernel<N, CP><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  const double macs = (double)sms * iters * 72 * 128.0 * N * 32.0;
  std::printf("%s N=%3d: %s  %.3f ms  %.1f TOP/s int8 dense (%.0f MAC/clk/SM at 1.92 GHz)\n", CP ? "TS+cp" : "TS", N,
              cudaGetErrorString(e), ms, 2 * macs / (ms * 1e-3) / 1e12,
              macs / sms / (ms * 1e-3) / 1.92e9);
  cudaFree(cyc);
}

// The split GEMM's issue order (TS): per 32-byte K step, for each A digit i
// one copy then the MMAs of pairs (i, j), i + j < 7, into accumulator i + j;
// 56 MMAs per commit (two K steps), as in oz_gemm_kernel.
// The 28 digit pairs (i, j) in an order that spreads the MMAs into each
// accumulator d = i + j (greedy: most remaining work among the longest idle).
__device__ __forceinline__ constexpr int kord(int q) {  // 8 i + j
  switch (q) {
    case 0: return 6;
    case 1: return 5;
    case 2: return 4;
    case 3: return 3;
    case 4: return 2;
    case 5: return 1;
    case 6: return 13;
    case 7: return 12;
    case 8: return 11;
    case 9: return 10;
    case 10: return 9;
    case 11: return 0;
    case 12: return 20;
    case 13: return 19;
    case 14: return 18;
    case 15: return 17;
    case 16: return 8;
    case 17: return 16;
    case 18: return 27;
    case 19: return 26;
    case 20: return 25;
    case 21: return 24;
    case 22: return 34;
    case 23: return 33;
    case 24: return 32;
    case 25: return 41;
    case 26: return 40;
    case 27: return 48;
  }
  return 0;
}
template <int MODE>  // 0: copy then MMAs per digit; 1: copies first, spread order; 2: copy one digit ahead
__global__ void __launch_bounds__(128, 1) order_kernel(int iters, unsigned long long* cycles) {
  constexpr bool GREEDY = MODE == 1;
  constexpr int N = 64;
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int bytes = 8 * (128 * 64) + 8 * (N * 64);
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  unsigned long long t0 = clock64();
  if (warp == 0) {
    const uint64_t ad0 = desc64(smem_u32(smem)), bd0 = desc64(smem_u32(smem + 8 * 128 * 64));
    uint32_t aslot = 0;
    for (int it = 0; it < iters; ++it) {
      if constexpr (MODE >= 2) {
        // A digit copies one digit ahead of their MMAs: (ks, i) -> slot aslot
        auto cp = [&](int ks, int i, uint32_t slot) {
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(tmem + (uint32_t)(7 * N + (slot & 7u) * 8u)),
              "l"(ad0 + (uint64_t)((i * 128 * 64 + ks * 32) >> 4)));
        };
        constexpr int AH = MODE == 3 ? 2 : 1;  // copy distance in digits (MODE 4: 1)
        if (it == 0)
          for (int a = 0; a < AH; ++a) cp(0, a, aslot + a);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
          for (int i = 0; i < 7; ++i, ++aslot) {
            const int q = ks * 7 + i + AH;  // digit index AH ahead, wrapping to the next batch
            cp((q / 7) & 1, q % 7, aslot + AH);
            const uint32_t ta = tmem + (uint32_t)(7 * N + (aslot & 7u) * 8u);
#pragma unroll
            for (int jj = 0; i + jj < 7; ++jj) {
              const int j = MODE == 4 ? 6 - i - jj : jj;  // MODE 4: accumulators high to low
              const uint64_t bd = bd0 + (uint64_t)((j * N * 64 + ks * 32) >> 4);
              asm volatile(
                  "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)((i + j) * N)),
                  "r"(ta), "l"(bd), "r"(idesc), "r"(1u));
            }
          }
        }
      } else
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        if constexpr (GREEDY) {
          const uint32_t base = aslot;
#pragma unroll
          for (int i = 0; i < 7; ++i, ++aslot)
            asm volatile(
                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(tmem + (uint32_t)(7 * N + (aslot & 7u) * 8u)),
                "l"(ad0 + (uint64_t)((i * 128 * 64 + ks * 32) >> 4)));
#pragma unroll
          for (int q = 0; q < 28; ++q) {
            constexpr int dummy = 0;
            (void)dummy;
            const int i = kord(q) >> 3, j = kord(q) & 7;
            const uint32_t ta = tmem + (uint32_t)(7 * N + ((base + i) & 7u) * 8u);
            const uint64_t bd = bd0 + (uint64_t)((j * N * 64 + ks * 32) >> 4);
            asm volatile(
                "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)((i + j) * N)),
                "r"(ta), "l"(bd), "r"(idesc), "r"(1u));
          }
          continue;
        }
#pragma unroll
        for (int i = 0; i < 7; ++i, ++aslot) {
          const uint32_t ta = tmem + (uint32_t)(7 * N + (aslot & 7u) * 8u);
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(ta),
              "l"(ad0 + (uint64_t)((i * 128 * 64 + ks * 32) >> 4)));
#pragma unroll
          for (int j = 0; i + j < 7; ++j) {
            const uint64_t bd = bd0 + (uint64_t)((j * N * 64 + ks * 32) >> 4);
            asm volatile(
                "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)((i + j) * N)),
                "r"(ta), "l"(bd), "r"(idesc), "r"(1u));
          }
        }
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
              smem_u32(&bar)));
      asm volatile(
          "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(
              smem_u32(&bar)), "r"((uint32_t)(it & 1)));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int MODE>
void run_order(int sms) {
  constexpr int N = 64;
  const int smem = 8 * 128 * 64 + 8 * N * 64 + 1024;
  cudaFuncSetAttribute(order_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  const int iters = 2000;
  order_kernel<MODE><<<sms, 128, smem>>>(10, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  order_kernel<MODE><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  const double macs = (double)sms * iters * 56 * 128.0 * N * 32.0;
  std::printf("%s N= 64: %s  %.3f ms  %.1f TOP/s int8 dense (%.0f MAC/clk/SM at 1.92 GHz)\n",
              MODE == 4 ? "split order, copy ahead, d high->low" : MODE == 3 ? "split order, copy 2 ahead" : MODE == 2 ? "split order, copy ahead" : MODE == 1 ? "split order, spread" : "split order",
              cudaGetErrorString(e), ms,
              2 * macs / (ms * 1e-3) / 1e12, macs / sms / (ms * 1e-3) / 1.92e9);
  cudaFree(cyc);
}

template <int N>
void run(int sms) {
  const int smem = 8 * 128 * 64 + 8 * N * 64 + 1024;
  cudaFuncSetAttribute(peak_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  const int iters = 2000;
  peak_kernel<N><<<sms, 128, smem>>>(10, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  peak_kernel<N><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  const double macs = (double)sms * iters * 72 * 128.0 * N * 32.0;
  std::printf("N=%3d: %s  %.3f ms  %.1f TOP/s int8 dense (%.0f MAC/clk/SM at 1.92 GHz)\n", N,
              cudaGetErrorString(e), ms, 2 * macs / (ms * 1e-3) / 1e12,
              macs / sms / (ms * 1e-3) / 1.92e9);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64>(sms);
  run_ts<64, false>(sms);
  run_ts<64, true>(sms);
  run_order<0>(sms);
  run_order<1>(sms);
  run_order<2>(sms);
  run_order<3>(sms);
  run_order<4>(sms);
  run<128>(sms);
  run<256>(sms);
  return 0;
}
