// Micro-probe of the per-SM limits the ping-pong attention runs into (bench-only, not part of libpic):
// cycles per tcgen05.mma (M=128, N=128, K=16, bf16) issued back to back by one thread, SS (A and B in
// smem) or TS (A in TMEM), alone and with 8 other warps streaming tcgen05.ld (LDTM) from other TMEM
// columns or ld.shared from smem, plus LDTM and MUFU.EX2 throughput alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_15332_b200/csrc/kernels \
//        scripts/probe_tc.cu -o build/probe_tc && build/probe_tc
#include <cstdio>
#include <cstdint>

#include "common.cuh"

using namespace pic;

__global__ void __launch_bounds__(320, 1) probe(int mode, int n_mma, int n_ld, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = smem_u32(smem);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool do_mma = mode & 1, ts = mode & 2, do_ldtm = mode & 4, do_lds = mode & 8, do_ex2 = mode & 16;
  const int nsel = (mode >> 8) & 3;  // 0: N=128, 1: N=64, 2: N=256
  const int nacc = (mode >> 10) & 3;   // independent accumulators cycled (0 -> 1)
  unsigned long long t0 = clock64();
  float acc = 0.f;
  if (warp == 1) {
    if (do_mma) {  // whole warp, elect.sync issue, descriptors precomputed, unrolled
      const uint32_t idS = nsel == 1 ? idesc_bf16(128, 64, 0, 0) : idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);
      const uint64_t dA = sdesc_sw128(base, 16, 1024), dB = sdesc_sw128(base + 32768, 16, 1024);
      const uint64_t dV = sdesc_sw128(base + 32768, 16384, 1024);
      const uint32_t d1 = nacc ? 128u : 0u, d1o = nacc ? 128u : 0u;
      for (int i = 0; i < n_mma; i += 16) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t o = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          if (ts) {
            umma_bf16_ts_e(tmem + 256, tmem + 384 + kk * 8, dV + (uint64_t)(kk * 128), idO, 1);
            umma_bf16_ts_e(tmem + 256 - d1o, tmem + 384 + kk * 8, dV + (uint64_t)(kk * 128), idO, 1);
          } else {
            umma_bf16_e(tmem + 0, dA + o, dB + o, idS, 1);
            umma_bf16_e(tmem + d1, dA + o, dB + o, idS, 1);
          }
        }
      }
      umma_commit_e(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
      if (lane == 0) out[blockIdx.x * 8 + 0] = clock64() - t0;
    }
  } else if (warp >= 2) {
    const int q = warp & 3;
    const uint32_t la = (uint32_t)(q * 32) << 16;
    if (do_ldtm) {
      for (int i = 0; i < n_ld; ++i) {
        float v[64];
        tmem_ld64(tmem + la + 128 + ((warp >> 2) & 1) * 64, v);
#pragma unroll
        for (int j = 0; j < 64; ++j) acc += v[j];
      }
    }
    if (do_lds) {
      for (int i = 0; i < n_ld; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint4 x = lds128(base + ((i * 16 + j) * 512 + lane * 16) % 65536);
          acc += __uint_as_float(x.x) + __uint_as_float(x.w);
        }
      }
    }
    if (do_ex2) {
      float x0 = lane * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
      for (int i = 0; i < n_ld; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          x0 = ex2_approx(x0 * -0.999f);
          x1 = ex2_approx(x1 * -0.999f);
          x2 = ex2_approx(x2 * -0.999f);
          x3 = ex2_approx(x3 * -0.999f);
        }
      }
      acc += x0 + x1 + x2 + x3;
    }
    if (lane == 0 && warp == 2) out[blockIdx.x * 8 + 1] = clock64() - t0;
  }
  if (acc == 12345.f) out[7] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const char* names[] = {"SS mma", "TS mma", "LDTM x64 (8 warps)", "SS mma + LDTM", "TS mma + LDTM", "LDS 128 (8 warps)",
                         "SS mma + LDS", "EX2 (8 warps, 4 chains, 64/iter)", "SS mma + EX2", "SS mma N=64", "SS mma 2 accumulators", "SS mma 3 accumulators", "TS mma 2 accumulators"};
  const int modes[] = {1, 3, 4, 5, 7, 8, 9, 16, 17, 1 | 256, 1 | 1024, 1 | 2048, 3 | 1024};
  const int n_mma = 8192, n_ld = 1024;
  for (int m = 0; m < 13; ++m) {
    cudaMemset(d, 0, 148 * 8 * 8);
    probe<<<148, 320, 65536 + 1024>>>(modes[m], n_mma, n_ld, d);
    probe<<<148, 320, 65536 + 1024>>>(modes[m], n_mma, n_ld, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[16];
    cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
    printf("%-32s err=%d  mma: %8.1f cyc/instr   other warps: %10llu cyc total (%6.1f cyc per iteration)\n", names[m],
           (int)e, h[0] ? (double)h[0] / n_mma : 0.0, h[1], h[1] ? (double)h[1] / n_ld : 0.0);
  }
  return 0;
}
