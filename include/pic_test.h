/*
 * pic_test.h — kernel-level test entry points of libpic.so (tests only; not part of the
 * product API).  Each runs ONE hot-path kernel on host-provided inputs through the same launcher
 * the engine uses, so GPU tests can localise a parity failure to a kernel.  All buffers are
 * host arrays; bf16 values are passed as uint16 bit patterns.  Device memory is cudaMalloc'ed and
 * freed inside the call.  Return pic_status as in pic.h.
 */
#ifndef PIC_TEST_H
#define PIC_TEST_H
#include "pic.h"

#ifdef __cplusplus
extern "C" {
#endif

/* tcgen05 GEMM (a5/a7/a8/a10): out[m][n] = Σ_k A[m][k]·B[n][k] (fp32, summed over `splits` split-K
 * partials), A [M][K], B [N][K] bf16; bn ∈ {64,128,256}; K % 64 == 0, N % 32 == 0.  A negative bn selects
 * the CTA-pair (cta_group::2, 256-row M-tile) kernel with N-tile |bn| ∈ {128,192,224,256} (also for
 * pic_test_gemm_swiglu and pic_bench_gemm). */
pic_status pic_test_gemm(const uint16_t* A, const uint16_t* B, int32_t M, int32_t N, int32_t K, int32_t bn,
                         int32_t splits, float* out);

/* tcgen05 GEMM with the fused SwiGLU epilogue (a8): B [N2][K] holds W_gate / W_up interleaved in groups of
 * bn/2 rows; u [M][N2/2] bf16 = silu(A·W_gᵀ) ⊙ (A·W_uᵀ). */
pic_status pic_test_gemm_swiglu(const uint16_t* A, const uint16_t* B, int32_t M, int32_t N2, int32_t K, int32_t bn,
                                uint16_t* u);

/* a6 sparse-query causal attention (tcgen05, D = 128) + split-KV combine over a PAGED copy of K/V:
 * K, V [n_keys][Hkv][128] bf16 are scattered into 16-token blocks in the order `block_perm`
 * (int32[ceil(n_keys/16)], a permutation of block ids < num_blocks), queries Q [M][Hq][128] at
 * positions pos[M] (sorted ascending, < n_keys), tiles of 128/G consecutive rows.  O [M][Hq][128] bf16. */
pic_status pic_test_attention(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* pos,
                              int32_t M, int32_t n_keys, int32_t Hq, int32_t Hkv, const int32_t* block_perm,
                              int32_t num_blocks, int32_t n_splits, uint16_t* O);

/* As pic_test_attention with the kernel chosen: version 1 = one q-tile per CTA (attention.cu), 2 = the
 * persistent ping-pong kernel (attention_pp.cu, the engine's default); grid > 0 caps the persistent grid
 * (several items per CTA), 0 = 148.  pic_test_attention = version 2, grid 0. */
pic_status pic_test_attention_v(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* pos,
                                int32_t M, int32_t n_keys, int32_t Hq, int32_t Hkv, const int32_t* block_perm,
                                int32_t num_blocks, int32_t n_splits, int32_t version, int32_t grid, uint16_t* O);

/* Engine-wide attention kernel override for later pic_link / pic_link_batch / pic_decode calls:
 * 0 = the engine's choice (default), 1 = one q-tile per CTA, 2 = ping-pong (also for shared-block links).
 * Tests and A/B measurements only. */
pic_status pic_test_set_attention_kernel(int32_t version);
/* The attention kernel the last forward launched (host-side record, set at launch or graph capture):
 * 1 one q-tile per CTA, 2 ping-pong, 3 chunk-frame one CTA per item, 4 chunk-frame persistent, 5 decode,
 * 6 SIMT (tiny head dims, fp32 debug build). */
int32_t pic_test_last_attention_kernel(void);

/* a2 KV link on a raw pool: pool K/V [n_layers][num_blocks][Hkv][16][D] bf16 (in/out), rows
 * (src_slot -> dst_slot, delta) for layers layer0..n_layers-1, RoPE table for positions < max_pos. */
pic_status pic_test_kv_link(uint16_t* Kpool, uint16_t* Vpool, int32_t n_layers, int32_t num_blocks, int32_t Hkv,
                            int32_t D, const int32_t* src_slot, const int32_t* dst_slot, const int32_t* delta,
                            int32_t n_rows, int32_t layer0, int32_t rebase, double theta, int32_t max_pos);

/* GEMM timing: average device µs per launch of the tcgen05 GEMM over `iters` back-to-back launches
 * (weights cycled through > 512 MB of copies so each launch streams from HBM). */
pic_status pic_bench_gemm(int32_t M, int32_t N, int32_t K, int32_t bn, int32_t splits, int32_t iters,
                          float* us_per_launch);

/* Attention timing: as pic_test_attention, then `iters` back-to-back launches of the attention
 * kernel alone; *us = average device µs per launch. */
pic_status pic_bench_attention(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* pos,
                               int32_t M, int32_t n_keys, int32_t Hq, int32_t Hkv, const int32_t* block_perm,
                               int32_t num_blocks, int32_t n_splits, int32_t iters, float* us);

#ifdef __cplusplus
}
#endif
#endif
