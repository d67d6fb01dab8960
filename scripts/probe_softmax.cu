// Micro-probe of the attention softmax step (bench-only, not part of libpic): per-SM throughput of
// MUFU.EX2 in its f32 / f16x2 / bf16x2 forms, and cycles per 128x128 S tile of the ping-pong kernel's
// register-resident softmax (row max, p = 2^(s*scale - m), row sum, bf16 pack) with 8 softmax warps per
// SM (two lanes x one warpgroup), for several exponential splits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_15332_b200/csrc/kernels \
//        scripts/probe_softmax.cu -o build/probe_softmax && build/probe_softmax
#include <cstdio>
#include <cstdint>

#include "common.cuh"

using namespace pic;

__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  uint32_t y;
  asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(y) : "f"(a), "f"(b));
  return y;
}

// raw MUFU throughput: 8 warps, 4 independent chains, 64 instructions per iteration per thread
template <int KIND>
__global__ void __launch_bounds__(256, 1) mufu_probe(int n_it, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  unsigned long long t0 = clock64();
  float acc = 0.f;
  if (KIND == 0) {
    float x0 = lane * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
    for (int i = 0; i < n_it; ++i) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        x0 = ex2_approx(x0 * -0.999f);
        x1 = ex2_approx(x1 * -0.999f);
        x2 = ex2_approx(x2 * -0.999f);
        x3 = ex2_approx(x3 * -0.999f);
      }
    }
    acc = x0 + x1 + x2 + x3;
  } else {
    uint32_t x0 = 0x3c003c00u + lane, x1 = x0 + 7, x2 = x0 + 13, x3 = x0 + 29;
    for (int i = 0; i < n_it; ++i) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        x0 = KIND == 1 ? ex2_f16x2(x0 ^ 0x80008000u) : ex2_bf16x2(x0 ^ 0x80008000u);
        x1 = KIND == 1 ? ex2_f16x2(x1 ^ 0x80008000u) : ex2_bf16x2(x1 ^ 0x80008000u);
        x2 = KIND == 1 ? ex2_f16x2(x2 ^ 0x80008000u) : ex2_bf16x2(x2 ^ 0x80008000u);
        x3 = KIND == 1 ? ex2_f16x2(x3 ^ 0x80008000u) : ex2_bf16x2(x3 ^ 0x80008000u);
      }
    }
    acc = __uint_as_float(x0 ^ x1 ^ x2 ^ x3);
  }
  const unsigned long long t = clock64() - t0;
  if (threadIdx.x == 0) out[blockIdx.x] = t;
  if (acc == 12345.f) out[1023] = 1;
}

// one softmax step per iteration: 128 scores per thread (one row of a 128x128 tile), 8 warps = 2 tiles
// VAR 0..3: f32 MUFU with VAR pairs of every 8 on the FMA-pipe polynomial; 4: bf16x2 MUFU (argument
// rounded to bf16, P comes out as bf16 pairs, row sum from the unpacked pairs); 5: f16x2 MUFU (argument
// rounded to f16, P converted to bf16 pairs)
template <int VAR>
__global__ void __launch_bounds__(256, 1) softmax_probe(int n_it, float sc, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  float v[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) v[i] = (float)((lane * 37 + i * 11) % 97) * 0.05f;
  uint32_t sink = 0;
  float l = 0.f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < n_it; ++it) {
    float m4[4] = {fmaxf(v[0], v[1]), fmaxf(v[2], v[3]), fmaxf(v[4], v[5]), fmaxf(v[6], v[7])};
#pragma unroll
    for (int i = 8; i < 128; i += 8) {
      m4[0] = fmax3(m4[0], v[i], v[i + 1]);
      m4[1] = fmax3(m4[1], v[i + 2], v[i + 3]);
      m4[2] = fmax3(m4[2], v[i + 4], v[i + 5]);
      m4[3] = fmax3(m4[3], v[i + 6], v[i + 7]);
    }
    const float m = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3])) + it * 1e-7f;
    const float2 nmu2 = make_float2(-m * sc, -m * sc), sc2 = make_float2(sc, sc);
    float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
    uint32_t pk[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const float2 xv = fma2(make_float2(v[2 * c], v[2 * c + 1]), sc2, nmu2);
      float2 pv;
      if constexpr (VAR <= 3) {
        if ((c & 7) < VAR)
          pv = exp2_poly2(xv);
        else
          pv = make_float2(ex2_approx(xv.x), ex2_approx(xv.y));
        pk[c] = pack_bf16(pv.x, pv.y);
      } else if constexpr (VAR == 4) {
        const uint32_t p = ex2_bf16x2(pack_bf16(xv.x, xv.y));
        pk[c] = p;
        pv = make_float2(__uint_as_float(p << 16), __uint_as_float(p & 0xFFFF0000u));
      } else {
        const uint32_t h = ex2_f16x2(pack_f16(xv.x, xv.y));
        __half2 hh = *reinterpret_cast<const __half2*>(&h);
        pv = __half22float2(hh);
        pk[c] = pack_bf16(pv.x, pv.y);
      }
      if (c & 1)
        lb = add2(lb, pv);
      else
        la = add2(la, pv);
    }
    l += (la.x + la.y) + (lb.x + lb.y);
#pragma unroll
    for (int c = 0; c < 64; ++c) sink ^= pk[c];
  }
  const unsigned long long t = clock64() - t0;
  if (threadIdx.x == 0) out[blockIdx.x] = t;
  if (sink == 12345u && l == 1.f) out[1023] = 1;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  const int n_it = 4096;
  auto run = [&](const char* name, void (*k)(int, unsigned long long*), double per_it_ops) {
    k<<<148, 256>>>(n_it, d);
    k<<<148, 256>>>(n_it, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-34s err=%d  %8.1f cyc/iter  %6.2f results/clk/SM\n", name, (int)e, (double)h / n_it,
           per_it_ops * 256 / ((double)h / n_it));
  };
  run("MUFU.EX2 f32", mufu_probe<0>, 64);
  run("MUFU.EX2 f16x2 (2 results/instr)", mufu_probe<1>, 128);
  run("MUFU.EX2 bf16x2 (2 results/instr)", mufu_probe<2>, 128);
  auto run_sm = [&](const char* name, void (*k)(int, float, unsigned long long*)) {
    const int it = 512;
    k<<<148, 256>>>(it, 0.127f, d);
    k<<<148, 256>>>(it, 0.127f, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    // one iteration = 8 warps x 32 rows x 128 keys = two 128x128 tiles
    printf("%-34s err=%d  %8.1f cyc per 128x128 tile\n", name, (int)e, (double)h / it / 2);
  };
  run_sm("softmax f32 MUFU, 0/8 poly", softmax_probe<0>);
  run_sm("softmax f32 MUFU, 1/8 poly", softmax_probe<1>);
  run_sm("softmax f32 MUFU, 2/8 poly", softmax_probe<2>);
  run_sm("softmax f32 MUFU, 3/8 poly", softmax_probe<3>);
  run_sm("softmax bf16x2 MUFU", softmax_probe<4>);
  run_sm("softmax f16x2 MUFU", softmax_probe<5>);
  return 0;
}
