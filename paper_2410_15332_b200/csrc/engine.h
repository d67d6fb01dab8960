// engine.h — internal state of a pic_engine (libpic.so).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../include/pic.h"
#include "kernels/kernels.h"

// Record a formatted message for pic_last_error() and return `s` (defined in engine.cpp).
pic_status pic_fail(pic_status s, const char* fmt, ...);

namespace pic {

// Deterministic paged-block allocator: lowest free ids first (D3; modelled by oracle.pic.BlockAllocator).
// Blocks are reference counted: a chunk-store block linked by reference (f3 shared-block link) is
// held by the store and by every live linked cache that points at it; it returns to the free list
// when the last holder releases it (expire_cache while a linked cache is live keeps it).
struct BlockAllocator {
  std::set<int32_t> free_ids;
  std::vector<int32_t> refs;
  void reset(int64_t n) {
    free_ids.clear();
    refs.assign(n, 0);
    for (int64_t i = 0; i < n; ++i) free_ids.insert(free_ids.end(), (int32_t)i);
  }
  void retain(int32_t b) { ++refs[b]; }
  bool can(int64_t n) const { return (int64_t)free_ids.size() >= n; }
  std::vector<int32_t> peek(int64_t n) const {
    std::vector<int32_t> v;
    for (auto it = free_ids.begin(); it != free_ids.end() && (int64_t)v.size() < n; ++it) v.push_back(*it);
    return v;
  }
  std::vector<int32_t> alloc(int64_t n) {
    std::vector<int32_t> v = peek(n);
    for (int32_t b : v) {
      free_ids.erase(b);
      refs[b] = 1;
    }
    return v;
  }
  void release(const std::vector<int32_t>& v) {
    for (int32_t b : v)
      if (--refs[b] == 0) free_ids.insert(b);
  }
};

struct ChunkRec {
  std::vector<int32_t> tokens;
  std::vector<int32_t> blocks;
  int32_t c0 = 0;  // compile position of row 0 (0; LegoLink-0 would use the dummy-prefix length)
};

struct LayerW {
  void *qkv, *o, *gu, *down;  // bf16 [out][in]
  float *g1, *g2;
  CUtensorMap tm_qkv[3], tm_o[3], tm_gu[3], tm_down[3];  // per GEMM N-tile (64/128/256)
  CUtensorMap tm_gu_fused;                                 // interleaved gate/up, box 2g rows (fused SwiGLU)
};

// One forward over a set of rows (a compile batch, one link or a batched link).
struct Fwd {
  int M = 0;                                  // rows recomputed at layer 0
  std::vector<int32_t> tok, pos, slot, seq;   // per row
  std::vector<int32_t> tiles;                 // attention q-tiles: (seq, row_start, row_count)
  std::vector<int32_t> seq_bt_off, bt;        // block tables (concatenated)
  std::vector<int32_t> bdelta;                // per bt entry: Δ still to apply to a shared block's keys (f3)
  bool kv_rot = false;                        // some bdelta != 0: attention re-bases K tiles on load
  std::vector<int32_t> kpos;                  // per row: RoPE position of its K heads (kv_share 3 chunk frames)
  bool has_kpos = false;
  bool attn_qrot = false;                     // attention re-bases by rotating Q per uniform-frame K tile
  bool qrot_ok = false;                       // kv_share 3 link: the Q-side re-base may apply
  std::vector<int32_t> vbt;                   // per bt entry: V's block (kv_share 2: the chunk-store block)
  bool has_vbt = false;                       // some vbt entry differs from bt
  std::vector<int32_t> k2_src, k2_dst, k2_delta;  // a2 work: cached rows gathered into linked blocks
  std::vector<int32_t> k2_vcopy;              // per a2 row: 1 = copy V too, 0 = K only (V by reference)
  bool k2_konly = false;                      // some a2 row copies K only
  int k2_layer0 = 0;
  std::vector<int32_t> head_map;              // per final row: request index or -1
  int n_head = 0;                             // requests producing logits (0 = compile)
  bool compile = false;
  int rebase = 1;
  int debug_rows = 0;                         // row stride of the debug_hidden capture (N)
  // CacheBlend (single request)
  bool cb = false;
  int cb_layer = 1, cb_T = 0, M2 = 0;
  bool cb_override = false;
  std::vector<int32_t> cb_cand, cb_forced, cb_sel2, cb_pos2, cb_slot2, tiles2, head_map2;
  // attention split-KV schedules (main rows, and CacheBlend rows after the check)
  std::vector<int32_t> attn_work, attn_nsplit, attn_work2, attn_nsplit2;
  int attn_n_work = 0, attn_n_work2 = 0, attn_max_split = 1, attn_max_split2 = 1;
  bool attn_pp = false;  // schedules in the ping-pong kernel's item format (attention_pp.cu)
  bool decode = false;       // pic_decode: one query row per sequence
  bool attn_decode = false;  // attention runs the split-KV decode kernel (attention_decode.cu)
};

// Per-request link bookkeeping produced by the planner.
struct ProfRec {
  std::string name;
  cudaEvent_t begin, end;
  double bytes, flops;
};
struct ProfAgg {
  int64_t launches = 0;
  double ms = 0, bytes = 0, flops = 0;
};

struct LinkPlanHost {
  int N = 0;
  std::vector<int32_t> tok;
  std::vector<int32_t> src_cid, src_row;       // -1 for dynamic rows
  std::vector<int32_t> chunk_start, chunk_len, chunk_delta;
  std::vector<uint64_t> chunk_id;
  std::vector<uint8_t> dynamic;
  std::vector<int32_t> sel;                    // sorted selected rows (pre-CacheBlend: dynamic ∪ {N-1})
};

}  // namespace pic

struct pic_linked {
  int32_t n_tokens = 0;
  std::vector<int32_t> blocks;
  std::vector<int32_t> bdelta;  // per block: Δ of a chunk-store block linked by reference (f3), or of an owned
                                // block kept in its chunk's compile frame (kv_share 3), else 0
  std::vector<uint8_t> byref;   // per block: 1 = blocks[b] is a chunk-store block linked by reference
  int32_t n_shared = 0;         // blocks linked by reference
  // kv_share 2: per block, the block holding its V rows — the chunk-store block (referenced, V by reference)
  // or blocks[b]; empty = blocks
  std::vector<int32_t> vblocks;
  int32_t n_vshared = 0;        // blocks whose V is linked by reference
};

struct pic_engine {
  pic_model_config cfg{};   // this rank's (local) model: heads / ffn_dim divided by tp_size
  pic_model_config gcfg{};  // global model
  int tp_rank = 0, tp_size = 1;
  bool f32 = false;         // fp32 debug build (dtype 1): fp32 activations / KV, CUDA-core GEMM + attention
  bool tp_connected = false;
  float* ar_buf[2] = {nullptr, nullptr};       // reduced partials exchanged across ranks (alternating)
  long long *tp_flags = nullptr, *tp_counter = nullptr;
  unsigned* attn_ctr = nullptr;   // 2 self-resetting counters of the persistent attention's item queue
  unsigned* chain_bar = nullptr;  // 2 self-resetting counters of the persistent GEMM chain's grid barrier
  float* peer_ar[2][8];                        // every rank's ar_buf (peer memory), own included
  pic::Peers peer_flags{};
  std::vector<void*> ipc_opened;
  int ar_parity = 0;
  pic_engine_limits lim{};
  int device = -1;
  bool host_only = true;
  int max_seqs = 0, max_tiles = 0, max_bt = 0, max_k2 = 0;
  int gu_group = 0;  // gate/up interleave group g (fused SwiGLU GEMM, N-tile 2g); 0 = separate SwiGLU kernel
  // arena
  char* arena = nullptr;
  size_t arena_bytes = 0;
  // weights
  std::vector<pic::LayerW> layers;
  void *E = nullptr, *Wlm = nullptr;
  float* gf = nullptr;
  CUtensorMap tm_lm[3];
  float *cos_t = nullptr, *sin_t = nullptr;
  // paged KV pools [L][NB][Hkv][16][D] bf16
  void *Kpool = nullptr, *Vpool = nullptr;
  int64_t layer_stride = 0;  // elements per layer per pool
  CUtensorMap tm_K, tm_V, tm_K8, tm_V8;  // one-block and eight-block boxes
  // activations / workspaces
  float *h = nullptr, *h2 = nullptr, *ws = nullptr;
  float* ssq = nullptr;  // fused-norm row partials [max_rows][kSsqStride]
  size_t ws_floats = 0;
  void *x = nullptr, *Obuf = nullptr, *u = nullptr, *Q = nullptr, *x_last = nullptr;
  float *o_part = nullptr, *ml_part = nullptr;
  int attn_rows_cap = 0;  // max splits*M of the attention partials
  float* logits = nullptr;
  int32_t* amax = nullptr;
  float* cb_dev = nullptr;
  CUtensorMap tm_x, tm_O, tm_u, tm_xlast, tm_Q;  // A operands (128-row boxes), Q (attention)
  // plan buffers
  int32_t* plan_dev = nullptr;
  int32_t* plan_host = nullptr;  // pinned staging
  size_t plan_cap_ints = 0;
  cudaEvent_t plan_ev = nullptr;
  float* host_logits = nullptr;  // pinned
  int32_t* host_amax = nullptr;  // pinned
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t side_stream = nullptr;   // a2 layers >= 1 overlap the first layers (joined before their attention)
  cudaEvent_t k2_fork = nullptr, k2_join = nullptr;
  std::vector<cudaEvent_t> k2_layer_done;  // per layer: the side-stream a2 of that layer landed
  int32_t* last_cb_sel2 = nullptr;  // device: CacheBlend selection of the last forward
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_pool_next = 0;
  std::vector<pic::ProfRec> prof_pending;
  std::map<std::string, pic::ProfAgg> prof_agg;
  // store
  std::map<pic_cache_id, pic::ChunkRec> store;
  uint64_t next_id = 1;
  pic::BlockAllocator alloc;
  // graphs
  std::map<std::vector<int64_t>, cudaGraphExec_t> graphs;
  std::map<std::pair<const void*, int>, CUtensorMap> wmaps;  // weight tensor maps for N-tiles other than 64/128/256
  // stats
  int64_t kernels_last = 0, h2d_last = 0, d2h_last = 0;
};
