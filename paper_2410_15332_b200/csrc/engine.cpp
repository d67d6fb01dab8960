// engine.cpp — the C ABI of libpic.so (include/pic.h): engine/arena setup, weight generation,
// chunk store + block allocator, the link planner (step a1), and the per-layer launch sequence
// of the linked-prefill forward (steps a2-a10), replayed through per-shape CUDA graphs.
#include "engine.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <cstdlib>
#include <unistd.h>

using namespace pic;

// ============================================================================ errors
static thread_local std::string g_err;

static pic_status vfail(pic_status s, const char* fmt, va_list ap) {
  char buf[1024];
  vsnprintf(buf, sizeof buf, fmt, ap);
  g_err = buf;
  return s;
}

static pic_status fail(pic_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfail(s, fmt, ap);
  va_end(ap);
  return s;
}

// Same error path for the other translation units (serve.cpp): sets pic_last_error().
pic_status pic_fail(pic_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfail(s, fmt, ap);
  va_end(ap);
  return s;
}

#define CK(expr)                                                                                                  \
  do {                                                                                                            \
    cudaError_t e_ = (expr);                                                                                      \
    if (e_ != cudaSuccess) return fail(PIC_E_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                                       __LINE__);                                                                 \
  } while (0)

// PIC_DEBUG_SYNC=1: synchronise after every launch with a 20 s deadline and name a hung or
// faulting kernel on stderr (debugging aid; graphs are disabled in this mode).
static bool debug_sync() {
  static int v = -1;
  if (v < 0) v = getenv("PIC_DEBUG_SYNC") ? 1 : 0;
  return v == 1;
}

static void dbg_sync(const char* what, cudaStream_t st) {
  if (!debug_sync()) return;
  char name[64];
  snprintf(name, sizeof name, "%s", what);
  if (char* p = strchr(name, '(')) *p = 0;
  for (int i = 0; i < 20000; ++i) {
    cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) {
      fprintf(stderr, "[pic] ok   %s\n", name);
      return;
    }
    if (e != cudaErrorNotReady) {
      fprintf(stderr, "[pic] FAIL %s: %s\n", name, cudaGetErrorString(e));
      fflush(stderr);
      _exit(4);
    }
    usleep(1000);
  }
  fprintf(stderr, "[pic] HANG %s\n", name);
  fflush(stderr);
  _exit(3);
}

#define CKL(expr)            \
  do {                       \
    CK(expr);                \
    dbg_sync(#expr, st);     \
  } while (0)

// Profiling (pic_set_profiling): CUDA events around every launch on the launching stream, tagged
// with the kernel class and its algorithmic bytes / FLOPs (SURVEY §8(d) formulas).
static pic_status prof_push(pic_engine* e, cudaStream_t st, const char* name, double bytes, double flops, bool begin);

// Bench-only timing ablation (PIC_ABLATE bit mask; results are wrong when set): skip every launch of
// a kernel class to measure its in-graph cost.  Never set by the engine, tests or bench.py.
// Bench-only attention timeline (PIC_ATTN_TRACE=1): every attention launch writes per-CTA timestamps
// into one static buffer (the last layer's launch wins); pic_link prints a summary after the call.
static int g_attn_trace_ctas = 0;
static unsigned long long* attn_trace_buffer() {
  static unsigned long long* buf = nullptr;
  static const bool on = getenv("PIC_ATTN_TRACE") != nullptr;
  if (on && !buf && cudaMalloc(&buf, 32 * 8192 * sizeof(unsigned long long)) != cudaSuccess) buf = nullptr;
  return on ? buf : nullptr;
}
// ping-pong kernel (attention_pp.cu): per-CTA cycle accounting, 32 counters per CTA
static void attn_pp_trace_print(int n_cta) {
  unsigned long long* buf = attn_trace_buffer();
  if (!buf || n_cta <= 0) return;
  std::vector<unsigned long long> t((size_t)32 * n_cta);
  if (cudaMemcpy(t.data(), buf, t.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  static const char* nm[23] = {"start", "end", "prod wait K-empty", "prod wait V-empty", "prod wait Q-empty", "prod tiles",
                               "mma wait K", "mma wait P", "mma wait V", "mma wait Q", "mma wait O-free",
                               "smA wait S", "smA compute", "smA epilogue", "smA steps", "smB wait S", "smB compute",
                               "smB epilogue", "smB steps", "rot wait K", "rot compute", "items", "-"};
  std::vector<double> span;
  for (int c = 0; c < n_cta; ++c) span.push_back((double)(t[32 * c + 1] - t[32 * c]));
  std::sort(span.begin(), span.end());
  fprintf(stderr, "  attn_pp CTA span (cycles): min %.0f med %.0f max %.0f\n", span[0], span[span.size() / 2], span.back());
  for (int k = 2; k < 22; ++k) {
    std::vector<double> v;
    for (int c = 0; c < n_cta; ++c) v.push_back((double)t[32 * c + k]);
    std::sort(v.begin(), v.end());
    fprintf(stderr, "  attn_pp %-18s min %10.0f med %10.0f max %10.0f (%.1f%% of median span)\n", nm[k], v[0],
            v[v.size() / 2], v.back(), 100.0 * v[v.size() / 2] / span[span.size() / 2]);
  }
}
static bool g_attn_trace_pp = false;

static void attn_trace_print(int n_cta) {
  if (g_attn_trace_pp) {
    attn_pp_trace_print(n_cta);
    return;
  }
  unsigned long long* buf = attn_trace_buffer();
  if (!buf || n_cta <= 0) return;
  std::vector<unsigned long long> t((size_t)32 * n_cta);
  if (cudaMemcpy(t.data(), buf, t.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < n_cta; ++c) t0 = std::min(t0, t[32 * c]);
  static const char* nm[8] = {"entry", "wait_done", "q_full", "first_S", "last_P", "last_O", "epi_done", "exit"};
  {
    std::vector<int> nt;
    for (int c = 0; c < n_cta; ++c) nt.push_back((int)t[32 * c + 7]);
    std::sort(nt.begin(), nt.end());
    fprintf(stderr, "  attn kv tiles per CTA: min %d med %d max %d\n", nt[0], nt[nt.size() / 2], nt.back());
  }
  {
    static const char* an[7] = {"wait S", "max+xchg", "exp+P", "mma wK", "mma wP", "mma wV", "mma wQd"};
    for (int k = 0; k < 7; ++k) {
      std::vector<double> v;
      for (int c = 0; c < n_cta; ++c)
        if (t[32 * c + 7] > 0) v.push_back((double)t[32 * c + 8 + k] / 1e3 / (double)t[32 * c + 7]);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      fprintf(stderr, "  attn per-tile %-9s min %6.3f med %6.3f max %6.3f us\n", an[k], v[0], v[v.size() / 2], v.back());
    }
  }
  {
    long fr = 0;  // QROT: chunk frames per CTA (one R(-Δ)·Q rotation each)
    for (int c = 0; c < n_cta; ++c) fr += (long)t[32 * c + 15];
    if (fr) fprintf(stderr, "  attn QROT frames per CTA: mean %.2f\n", (double)fr / n_cta);
    static const char* pn[7] = {"S load", "max", "xchg", "rescale", "exp", "P store", "o_full+arrive"};
    double ph[7] = {0, 0, 0, 0, 0, 0, 0}, nt = 0;
    for (int c = 0; c < n_cta; ++c) {
      nt += (double)t[32 * c + 7];
      for (int k = 0; k < 7; ++k) ph[k] += (double)t[32 * c + 16 + k];
    }
    if (nt > 0) {
      fprintf(stderr, "  attn softmax cycles per tile (warp 2):");
      for (int k = 0; k < 7; ++k) fprintf(stderr, " %s %.0f", pn[k], ph[k] / nt);
      fprintf(stderr, "\n");
    }
    double ml = 0, mn = 0;
    for (int c = 0; c < n_cta; ++c) {
      ml += (double)t[32 * c + 23];
      mn += (double)t[32 * c + 24];
    }
    if (mn > 0) fprintf(stderr, "  attn P(t-1) arrive -> S(t+1) ready: %.0f cycles (PV + S = 16 MMAs)\n", ml / mn);
    double sw = 0, sr = 0, sa = 0;
    for (int c = 0; c < n_cta; ++c) {
      sw += (double)t[32 * c + 25];
      sr += (double)t[32 * c + 26];
      sa += (double)t[32 * c + 27];
    }
    if (mn > 0)
      fprintf(stderr, "  attn   = warp-2 arrive -> MMA warp sees P %.0f + MMA warp sees P -> S(t+1) ready %.0f cycles\n",
              (sw - sa) / mn, (sr - sw) / mn);
    // CTA span (entry -> exit) and its parts, summed over CTAs, per KV tile
    double sp = 0, pro = 0, epi = 0, tiles = 0;
    for (int c = 0; c < n_cta; ++c) {
      const unsigned long long* x = &t[32 * c];
      if (!x[7] || x[3] < x[0] || x[6] < x[3] || x[7] < x[0]) continue;
      sp += (double)(x[6] - x[0]);
      pro += (double)(x[3] - x[0]);
      epi += (double)(x[6] - x[5]);
      tiles += (double)x[7];
    }
    if (tiles > 0)
      fprintf(stderr, "  attn per KV tile (sum over CTAs): entry->epi_done %.3f us = prologue %.3f + loop %.3f + epilogue %.3f\n",
              sp / tiles / 1e3, pro / tiles / 1e3, (sp - pro - epi) / tiles / 1e3, epi / tiles / 1e3);
  }
  for (int k = 0; k < 7; ++k) {
    std::vector<double> v;
    for (int c = 0; c < n_cta; ++c)
      if (t[32 * c + k] >= t0) v.push_back((double)(t[32 * c + k] - t0) / 1e3);
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    fprintf(stderr, "  attn %-9s min %7.2f  med %7.2f  max %7.2f us (n=%zu)\n", nm[k], v[0], v[v.size() / 2], v.back(),
            v.size());
  }
}

// Bench-only chain timeline (PIC_CHAIN_TRACE=1): per layer and CTA: entry, per phase boundary
// (epilogue done, barrier passed), exit.  pic_link prints the middle layer.
static unsigned long long* chain_trace_buffer() {
  static unsigned long long* buf = nullptr;
  static const bool on = getenv("PIC_CHAIN_TRACE") != nullptr;
  if (on && !buf && cudaMalloc(&buf, (size_t)16 * 148 * 128 * sizeof(unsigned long long)) != cudaSuccess) buf = nullptr;
  return on ? buf : nullptr;
}
static void chain_trace_dump(int layer) {
  unsigned long long* buf = chain_trace_buffer();
  if (!buf) return;
  std::vector<unsigned long long> t(16 * 148);
  if (cudaMemcpy(t.data(), buf + (size_t)layer * 16 * 148, t.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < 148; ++c)
    if (t[16 * c]) t0 = std::min(t0, t[16 * c]);
  for (int k = 0; k < 16; ++k) {
    std::vector<double> v;
    for (int c = 0; c < 148; ++c)
      if (t[16 * c + k] >= t0 && t[16 * c + k]) v.push_back((double)(t[16 * c + k] - t0) / 1e3);
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    fprintf(stderr, "  chain L%d slot %2d min %7.2f  med %7.2f  max %7.2f us (n=%zu)\n", layer, k, v[0], v[v.size() / 2],
            v.back(), v.size());
  }
}

// The persistent GEMM chain is opt-in (PIC_CHAIN=1): measured on cfg2 it streams each phase at the
// same rate as the separate kernels, and its norm phases and grid barriers add ~18 µs per layer
// (4.77 vs 4.28 ms per link), so the separate PDL-chained kernels remain the default.
// a2 on a side stream overlapping the projections (PIC_K2_OVERLAP=1).  Off by default: measured at cfg4
// (copy path, 32-request waves) the co-running copy kernels slow the tensor-bound GEMMs more than they
// save — 949 ms per step with a2 on the main stream vs 999 with per-layer side-stream launches.
static bool k2_overlap() {
  static const bool on = getenv("PIC_K2_OVERLAP") != nullptr;
  return on;
}

// Consumers fused into unsplit GEMM epilogues (a5 RoPE + scatter, a7/a8 residual add); PIC_NO_EPI_FUSE=1
// keeps the separate kernels (A/B and the bit-identity test only)
static bool epi_fuse() {
  static const bool on = getenv("PIC_NO_EPI_FUSE") == nullptr;
  return on;
}
// Wave-quantised N-tile choice for multi-m-tile GEMMs (PIC_NO_WAVE_FIT=1: the bn 128/256 rule only)
static bool wave_fit() {
  static const bool on = getenv("PIC_NO_WAVE_FIT") == nullptr;
  return on;
}

// test hook: 0 = the engine's choice, 1 / 2 = force the one-lane / ping-pong attention kernel
namespace pic {
int g_attn_force = 0;
// test hook: the attention kernel the last forward launched (1 one-lane, 2 ping-pong, 3 one-CTA chunk-frame,
// 4 persistent chunk-frame, 5 decode, 6 SIMT) — set on the host at launch (or graph capture)
int g_attn_last_kind = 0;
}
// a6 on the persistent ping-pong kernel (attention_pp.cu); PIC_ATTN_V1=1: the one-lane kernel (A/B only)
static bool attn_pp_enabled() {
  static const bool on = getenv("PIC_ATTN_V1") == nullptr;
  return on;
}

// a4 RMSNorm fused across unsplit GEMM boundaries (residual epilogue writes bf16(h·g) + Σh² partials, the
// consumer's epilogue applies the row scale); PIC_NO_NORM_FUSE=1 keeps the residual_rmsnorm kernel
static bool norm_fuse() {
  static const bool on = getenv("PIC_NO_NORM_FUSE") == nullptr;
  return on;
}

static bool chain_enabled() {
  static const bool on = getenv("PIC_CHAIN") != nullptr;
  return on;
}

static bool ablated(const char* name) {
  static const int mask = getenv("PIC_ABLATE") ? atoi(getenv("PIC_ABLATE")) : 0;
  if (!mask) return false;
  static const char* names[] = {"rmsnorm", "qkv_rope_scatter", "attention", "attn_combine", "gemm", "kv_link", "swiglu"};
  for (int i = 0; i < 7; ++i)
    if ((mask >> i & 1) && !strcmp(name, names[i])) return true;
  return false;
}

#define PROF(name, bytes, flops, expr)                                      \
  do {                                                                      \
    if (e->profiling) TRY(prof_push(e, st, name, bytes, flops, true));      \
    if (!ablated(name)) CKL(expr);                                          \
    if (e->profiling) TRY(prof_push(e, st, name, 0, 0, false));             \
  } while (0)

#define TRY(expr)                    \
  do {                               \
    pic_status s_ = (expr);          \
    if (s_ != PIC_OK) return s_;     \
  } while (0)

extern "C" const char* pic_last_error(void) { return g_err.c_str(); }

extern "C" const char* pic_status_string(pic_status s) {
  switch (s) {
    case PIC_OK: return "PIC_OK";
    case PIC_E_INVALID_ARG: return "PIC_E_INVALID_ARG";
    case PIC_E_CONFIG: return "PIC_E_CONFIG";
    case PIC_E_EMPTY_INPUT: return "PIC_E_EMPTY_INPUT";
    case PIC_E_CAPACITY: return "PIC_E_CAPACITY";
    case PIC_E_MISSING_CACHE: return "PIC_E_MISSING_CACHE";
    case PIC_E_LAYOUT: return "PIC_E_LAYOUT";
    case PIC_E_VARIANT: return "PIC_E_VARIANT";
    case PIC_E_OOM: return "PIC_E_OOM";
    case PIC_E_CUDA: return "PIC_E_CUDA";
    case PIC_E_NO_DEVICE: return "PIC_E_NO_DEVICE";
    case PIC_E_TOKEN: return "PIC_E_TOKEN";
  }
  return "PIC_E_?";
}

// ============================================================================ config / arena
static const int kBN[3] = {64, 128, 256};

static pic_status validate_cfg(const pic_model_config* c, const pic_engine_limits* l) {
  if (!c || !l) return fail(PIC_E_INVALID_ARG, "NULL config or limits");
  if (c->n_layers <= 0 || c->d_model <= 0 || c->n_heads <= 0 || c->n_kv_heads <= 0 || c->head_dim <= 0 ||
      c->ffn_dim <= 0 || c->vocab <= 0 || c->max_pos <= 0)
    return fail(PIC_E_CONFIG, "non-positive model dimension");
  if (c->n_heads % c->n_kv_heads) return fail(PIC_E_CONFIG, "n_heads %% n_kv_heads != 0");
  const int G = c->n_heads / c->n_kv_heads;
  if (128 % G) return fail(PIC_E_CONFIG, "GQA group %d must divide 128", G);
  if (c->head_dim != 16 && c->head_dim != 32 && c->head_dim != 64 && c->head_dim != 128)
    return fail(PIC_E_CONFIG, "head_dim must be 16/32/64/128");
  if (c->d_model % 64 || c->ffn_dim % 64 || (c->n_heads * c->head_dim) % 64)
    return fail(PIC_E_CONFIG, "d_model, ffn_dim, n_heads*head_dim must be multiples of 64");
  if (c->vocab % 32) return fail(PIC_E_CONFIG, "vocab must be a multiple of 32");
  if (c->dtype != 0 && c->dtype != 1) return fail(PIC_E_CONFIG, "dtype must be 0 (bf16) or 1 (fp32 debug)");
  if (c->bos_id < 0 || c->bos_id >= c->vocab) return fail(PIC_E_CONFIG, "bos_id out of range");
  if (!(c->rope_theta > 1.0) || !(c->rms_eps > 0.0)) return fail(PIC_E_CONFIG, "bad rope_theta / rms_eps");
  if (l->num_blocks <= 0 || l->max_rows <= 0 || l->max_tokens <= 0 || l->max_requests <= 0)
    return fail(PIC_E_INVALID_ARG, "non-positive limits");
  if (l->max_tokens > c->max_pos) return fail(PIC_E_CONFIG, "max_tokens > max_pos");
  if (l->num_blocks >= (1ll << 27)) return fail(PIC_E_CONFIG, "num_blocks too large for int32 slots");
  return PIC_OK;
}

struct Layout {
  size_t total = 0;
  std::vector<std::pair<void**, size_t>> items;
  size_t add(size_t bytes) {
    size_t off = (total + 1023) & ~size_t(1023);
    total = off + bytes;
    return off;
  }
};

struct ArenaPlan {
  size_t w_qkv, w_o, w_gu, w_down, w_g;  // per layer sizes
  size_t off_layers, layer_bytes;
  size_t off_E, off_lm, off_gf, off_cos, off_sin, off_K, off_V;
  size_t off_ssq;
  size_t off_h, off_h2, off_ws, off_x, off_O, off_u, off_Q, off_xlast, off_opart, off_ml, off_logits, off_amax,
      off_cbdev, off_plan;
  size_t off_ar, off_tpflags;
  size_t ws_floats;
  int attn_rows_cap, max_seqs, max_tiles, max_bt, max_k2;
  size_t plan_ints;
  size_t total;
};

static ArenaPlan plan_arena(const pic_model_config& c, const pic_engine_limits& l) {
  ArenaPlan a{};
  const size_t d = c.d_model, D = c.head_dim, Hq = c.n_heads, Hkv = c.n_kv_heads, F = c.ffn_dim, V = c.vocab;
  const size_t qkv = (Hq + 2 * Hkv) * D;
  Layout L;
  a.w_qkv = qkv * d * 2;
  a.w_o = d * Hq * D * 2;
  a.w_gu = 2 * F * d * 2;
  a.w_down = d * F * 2;
  a.w_g = d * 4;
  auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  a.layer_bytes = al(a.w_qkv) + al(a.w_o) + al(a.w_gu) + al(a.w_down) + 2 * al(a.w_g);
  a.off_layers = L.add(a.layer_bytes * c.n_layers);
  a.off_E = L.add(V * d * 2);
  a.off_lm = L.add(V * d * 2);
  a.off_gf = L.add(d * 4);
  a.off_cos = L.add((size_t)c.max_pos * (D / 2) * 4);
  a.off_sin = L.add((size_t)c.max_pos * (D / 2) * 4);
  const size_t es = c.dtype == 1 ? 4 : 2;  // activation / KV element size (fp32 debug build: 4)
  const size_t pool = (size_t)c.n_layers * l.num_blocks * Hkv * 16 * D * es;
  a.off_K = L.add(pool);
  a.off_V = L.add(pool);
  const size_t M = l.max_rows;
  a.off_h = L.add(M * d * 4);
  a.off_h2 = L.add(M * d * 4);
  a.off_ssq = L.add(M * kSsqStride * 4);  // fused-norm row partials (Σ h² per n-tile)
  size_t wsf = std::max({M * qkv, M * 2 * F, M * d, (size_t)l.max_requests * V});
  wsf = std::max(wsf, (size_t)148 * 128 * 256 * 2);
  a.ws_floats = wsf;
  a.off_ws = L.add(wsf * 4);
  a.off_x = L.add(M * std::max(d, Hq * D) * es);
  a.off_O = L.add(M * Hq * D * es);
  a.off_u = L.add(M * F * es);
  a.off_Q = L.add(M * Hq * D * es);
  a.off_xlast = L.add((size_t)l.max_requests * d * es);
  a.attn_rows_cap = (int)std::max<size_t>(4 * M, 2048);
  a.off_opart = L.add((size_t)a.attn_rows_cap * Hq * 128 * 4);
  a.off_ml = L.add((size_t)a.attn_rows_cap * Hq * 2 * 4);
  a.off_logits = L.add((size_t)l.max_requests * V * 4);
  a.off_amax = L.add((size_t)l.max_requests * 4);
  a.off_cbdev = L.add((size_t)l.max_tokens * 4);
  a.max_seqs = std::max(l.max_requests, 256);
  a.max_tiles = l.max_rows + a.max_seqs;
  a.max_bt = (int)((size_t)l.max_requests * ((l.max_tokens + 15) / 16) + l.max_rows / 16 + a.max_seqs + 16);
  a.max_k2 = (int)std::min<size_t>((size_t)l.max_requests * l.max_tokens, (size_t)1 << 30);
  // per-row arrays (tok,pos,slot,seq,head) + tiles + seq offsets + bt + k2 (3) + CB (cand,forced,sel2,pos2,slot2,
  // keep,count) + tiles2 + head2
  a.plan_ints = 5 * M + 3 * (size_t)a.max_tiles + a.max_seqs + 3 * (size_t)a.max_bt /* bt, bdelta, vbt */ + 4 * (size_t)a.max_k2 +
                7 * (size_t)l.max_tokens + 8 * (size_t)a.max_tiles + M + 8192;  /* + attention items (8 ints) */
  a.off_plan = L.add(a.plan_ints * 4);
  // tensor parallel: two reduced-partial buffers (alternating per all-reduce), flags, epoch counter
  a.off_ar = L.add(2 * M * d * 4);
  a.off_tpflags = L.add(8 * 8 + 8 + 16 + 16);  // TP epoch flags + counter, GEMM-chain barrier, attention item counters
  a.total = L.total + 1024;
  return a;
}

// Per-rank model: heads and MLP columns sharded over tp ranks; d_model, vocab replicated.
static pic_model_config local_cfg(const pic_model_config& g, int tp) {
  pic_model_config c = g;
  c.n_heads /= tp;
  c.n_kv_heads /= tp;
  c.ffn_dim /= tp;
  return c;
}

static pic_status validate_tp(const pic_model_config* c, int tp_rank, int tp_size) {
  if (tp_size < 1 || tp_size > 8 || tp_rank < 0 || tp_rank >= tp_size)
    return fail(PIC_E_INVALID_ARG, "bad tensor-parallel rank %d / size %d (size 1..8)", tp_rank, tp_size);
  if (c->n_heads % tp_size || c->n_kv_heads % tp_size || c->ffn_dim % tp_size || (c->ffn_dim / tp_size) % 64)
    return fail(PIC_E_CONFIG, "heads / kv-heads / ffn_dim not divisible by tp %d (ffn_dim/tp %% 64)", tp_size);
  return PIC_OK;
}

extern "C" pic_status pic_arena_bytes(const pic_model_config* cfg, const pic_engine_limits* limits, size_t* out) {
  TRY(validate_cfg(cfg, limits));
  if (!out) return fail(PIC_E_INVALID_ARG, "NULL out_bytes");
  *out = plan_arena(*cfg, *limits).total;
  return PIC_OK;
}

extern "C" pic_status pic_arena_bytes_tp(const pic_model_config* cfg, const pic_engine_limits* limits, int32_t tp_size,
                                         size_t* out) {
  TRY(validate_cfg(cfg, limits));
  TRY(validate_tp(cfg, 0, tp_size));
  if (!out) return fail(PIC_E_INVALID_ARG, "NULL out_bytes");
  const pic_model_config lc = local_cfg(*cfg, tp_size);
  TRY(validate_cfg(&lc, limits));
  *out = plan_arena(lc, *limits).total;
  return PIC_OK;
}

// ============================================================================ tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static pic_status get_encoder() {
  if (g_encode) return PIC_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(PIC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return PIC_OK;
}

// bf16 tensor map, SWIZZLE_128B, dims[0] innermost; strides in bytes for dims 1..rank-1
static pic_status make_tmap(CUtensorMap* m, void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                            const uint32_t* box) {
  uint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PIC_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PIC_OK;
}

// row-major [rows][cols] bf16 matrix, box = 64 cols x box_rows rows
static pic_status make_tmap_2d(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  uint64_t dims[2] = {cols, rows};
  uint64_t strides[1] = {cols * 2};
  uint32_t box[2] = {64, box_rows};
  return make_tmap(m, base, 2, dims, strides, box);
}

static pic_status make_tmaps_bn(CUtensorMap* m3, void* base, uint64_t rows, uint64_t cols) {
  for (int i = 0; i < 3; ++i) TRY(make_tmap_2d(&m3[i], base, rows, cols, kBN[i]));
  return PIC_OK;
}

static int bn_index(int bn) { return bn == 64 ? 0 : (bn == 128 ? 1 : 2); }

// ============================================================================ engine create
static int weight_exponent(int64_t fan_in) { return (int)std::nearbyint(std::log2(std::sqrt(3.0 / (double)fan_in))); }

static pic_status init_device(pic_engine* e, void* arena, size_t bytes, cudaStream_t st) {
  const pic_model_config& c = e->cfg;
  const ArenaPlan a = plan_arena(c, e->lim);
  if (!arena) return fail(PIC_E_INVALID_ARG, "NULL arena for a device engine");
  if (bytes < a.total) return fail(PIC_E_LAYOUT, "arena too small: %zu < %zu bytes", bytes, a.total);
  if (reinterpret_cast<uintptr_t>(arena) & 255) return fail(PIC_E_LAYOUT, "arena not 256-byte aligned");
  TRY(get_encoder());
  char* b = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(arena) + 1023) & ~uintptr_t(1023));
  e->arena = b;
  e->arena_bytes = bytes;
  e->max_seqs = a.max_seqs;
  e->max_tiles = a.max_tiles;
  e->max_bt = a.max_bt;
  e->max_k2 = a.max_k2;
  const int64_t d = c.d_model, D = c.head_dim, Hq = c.n_heads, Hkv = c.n_kv_heads, F = c.ffn_dim, V = c.vocab;
  const int64_t qkv = (Hq + 2 * Hkv) * D;
  const uint64_t s = c.seed;
  auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  // tensor-parallel shard of the global weights: rank r owns q heads [r·Hq, (r+1)·Hq), kv heads
  // [r·Hkv, ...), MLP columns [r·F, (r+1)·F) (local sizes); exponents use the GLOBAL fan-in.
  const int64_t tr = e->tp_rank, tp = e->tp_size;
  const int64_t gHqD = Hq * D * tp, gF = F * tp;
  // gate/up interleave group for the fused SwiGLU epilogue (fixed when the weights are generated, so
  // before any M is known): the g dividing F that minimises waves x per-unit cost (2g + 64: an N-tile
  // of 2g weight rows plus the fixed A-tile / epilogue cost) summed over a skinny (1 m-tile) and a
  // wide (8 m-tiles, per m-tile) forward.  Mistral/Llama F = 14336 and Llama-70B F = 28672: g = 112
  // (N-tile 224; 128 tiles fill one wave at k' <= 128).  (A wave-fill-only rule picked g = 16 for
  // F = 28672: N-tile 32, 3.5x slower GEMMs at k' = 1072.)
  e->f32 = c.dtype == 1;
  e->gu_group = 0;
  if (!getenv("PIC_NO_FUSED_SWIGLU") && !e->f32) {
    double best = 1e300;
    for (int g : {112, 128, 64, 32, 16}) {
      if (F % g || !gemm_bn_supported(2 * g, true)) continue;
      const int64_t tiles = F / g;
      double cost = 0;
      for (int mt : {1, 8}) cost += (double)((mt * tiles + 147) / 148) * (2 * g + 64) / mt;
      if (cost < best - 1e-9) {
        best = cost;
        e->gu_group = g;
      }
    }
    if (const char* ge = getenv("PIC_GU_GROUP")) {  // A/B override of the interleave group
      const int g = atoi(ge);
      if (g > 0 && F % g == 0 && gemm_bn_supported(2 * g, true)) e->gu_group = g;
    }
  }
  e->layers.resize(c.n_layers);
  for (int l = 0; l < c.n_layers; ++l) {
    LayerW& w = e->layers[l];
    char* p = b + a.off_layers + (size_t)l * a.layer_bytes;
    w.qkv = p;
    p += al(a.w_qkv);
    w.o = p;
    p += al(a.w_o);
    w.gu = p;
    p += al(a.w_gu);
    w.down = p;
    p += al(a.w_down);
    w.g1 = reinterpret_cast<float*>(p);
    p += al(a.w_g);
    w.g2 = reinterpret_cast<float*>(p);
    const uint64_t T = (uint64_t)l * 16;
    char* q = reinterpret_cast<char*>(w.qkv);
    CK(launch_gen_matrix(q, Hq * D, d, s, T + 0, weight_exponent(d), tr * Hq * D, st));
    CK(launch_gen_matrix(q + Hq * D * d * 2, Hkv * D, d, s, T + 1, weight_exponent(d), tr * Hkv * D, st));
    CK(launch_gen_matrix(q + (Hq + Hkv) * D * d * 2, Hkv * D, d, s, T + 2, weight_exponent(d), tr * Hkv * D, st));
    CK(launch_gen_matrix(w.o, d, Hq * D, s, T + 3, weight_exponent(gHqD), 0, st, gHqD, tr * Hq * D));
    if (e->gu_group > 0) {
      // gate/up interleaved in groups of g rows for the fused SwiGLU GEMM epilogue
      CK(launch_gen_gateup(w.gu, F, d, s, T + 4, T + 5, weight_exponent(d), e->gu_group, st, tr * F));
    } else {
      char* gu = reinterpret_cast<char*>(w.gu);
      CK(launch_gen_matrix(gu, F, d, s, T + 4, weight_exponent(d), tr * F, st));
      CK(launch_gen_matrix(gu + F * d * 2, F, d, s, T + 5, weight_exponent(d), tr * F, st));
    }
    CK(launch_gen_matrix(w.down, d, F, s, T + 6, weight_exponent(gF), 0, st, gF, tr * F));
    CK(launch_gen_gains(w.g1, d, s, T + 7, st));
    CK(launch_gen_gains(w.g2, d, s, T + 8, st));
    TRY(make_tmaps_bn(w.tm_qkv, w.qkv, qkv, d));
    TRY(make_tmaps_bn(w.tm_o, w.o, d, Hq * D));
    if (e->gu_group > 0)
      TRY(make_tmap_2d(&w.tm_gu_fused, w.gu, 2 * F, d, 2 * e->gu_group));
    TRY(make_tmaps_bn(w.tm_gu, w.gu, 2 * F, d));
    TRY(make_tmaps_bn(w.tm_down, w.down, d, F));
  }
  e->E = b + a.off_E;
  e->Wlm = b + a.off_lm;
  e->gf = reinterpret_cast<float*>(b + a.off_gf);
  CK(launch_gen_matrix(e->E, V, d, s, 0xE0000001ull, 0, 0, st));
  CK(launch_gen_matrix(e->Wlm, V, d, s, 0xE0000002ull, weight_exponent(d), 0, st));
  CK(launch_gen_gains(e->gf, d, s, 0xE0000003ull, st));
  TRY(make_tmaps_bn(e->tm_lm, e->Wlm, V, d));

  // RoPE table: angle = p · θ^(−2j/D) in fp64, stored fp32 (reading R2)
  e->cos_t = reinterpret_cast<float*>(b + a.off_cos);
  e->sin_t = reinterpret_cast<float*>(b + a.off_sin);
  {
    const int64_t half = D / 2, n = (int64_t)c.max_pos * half;
    std::vector<float> cs(n), sn(n);
    std::vector<double> inv(half);
    for (int64_t j = 0; j < half; ++j) inv[j] = std::pow(c.rope_theta, -2.0 * (double)j / (double)D);
    for (int64_t p = 0; p < c.max_pos; ++p)
      for (int64_t j = 0; j < half; ++j) {
        const double ang = (double)p * inv[j];
        cs[p * half + j] = (float)std::cos(ang);
        sn[p * half + j] = (float)std::sin(ang);
      }
    CK(cudaMemcpyAsync(e->cos_t, cs.data(), n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(e->sin_t, sn.data(), n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }

  // paged pools, zeroed so never-written slots are finite (masked keys multiply P = 0)
  e->Kpool = b + a.off_K;
  e->Vpool = b + a.off_V;
  e->layer_stride = e->lim.num_blocks * Hkv * 16 * D;
  const size_t pool = (size_t)c.n_layers * e->layer_stride * (e->f32 ? 4 : 2);
  CK(cudaMemsetAsync(e->Kpool, 0, pool, st));
  CK(cudaMemsetAsync(e->Vpool, 0, pool, st));
  if (D >= 64 && !e->f32) {
    uint64_t dims[4] = {(uint64_t)D, 16, (uint64_t)Hkv, (uint64_t)c.n_layers * e->lim.num_blocks};
    uint64_t strides[3] = {(uint64_t)D * 2, (uint64_t)16 * D * 2, (uint64_t)Hkv * 16 * D * 2};
    uint32_t box[4] = {64, 16, 1, 1};
    TRY(make_tmap(&e->tm_K, e->Kpool, 4, dims, strides, box));
    TRY(make_tmap(&e->tm_V, e->Vpool, 4, dims, strides, box));
    uint32_t box8[4] = {64, 16, 1, 8};
    TRY(make_tmap(&e->tm_K8, e->Kpool, 4, dims, strides, box8));
    TRY(make_tmap(&e->tm_V8, e->Vpool, 4, dims, strides, box8));
  }
  const int64_t M = e->lim.max_rows;
  e->h = reinterpret_cast<float*>(b + a.off_h);
  e->h2 = reinterpret_cast<float*>(b + a.off_h2);
  e->ssq = reinterpret_cast<float*>(b + a.off_ssq);
  e->ws = reinterpret_cast<float*>(b + a.off_ws);
  e->ws_floats = a.ws_floats;
  e->x = b + a.off_x;
  e->Obuf = b + a.off_O;
  e->u = b + a.off_u;
  e->Q = b + a.off_Q;
  e->x_last = b + a.off_xlast;
  e->o_part = reinterpret_cast<float*>(b + a.off_opart);
  e->ml_part = reinterpret_cast<float*>(b + a.off_ml);
  e->attn_rows_cap = a.attn_rows_cap;
  e->logits = reinterpret_cast<float*>(b + a.off_logits);
  e->amax = reinterpret_cast<int32_t*>(b + a.off_amax);
  e->cb_dev = reinterpret_cast<float*>(b + a.off_cbdev);
  e->plan_dev = reinterpret_cast<int32_t*>(b + a.off_plan);
  e->plan_cap_ints = a.plan_ints;
  // A operands: the GEMM always stages 128-row A tiles
  TRY(make_tmap_2d(&e->tm_x, e->x, M, d, 128));
  TRY(make_tmap_2d(&e->tm_O, e->Obuf, M, Hq * D, 128));
  TRY(make_tmap_2d(&e->tm_u, e->u, M, F, 128));
  TRY(make_tmap_2d(&e->tm_xlast, e->x_last, e->lim.max_requests, d, 128));
  if (D == 128 && !e->f32) {
    const int G = (int)(Hq / Hkv);
    uint64_t dims[3] = {(uint64_t)D, (uint64_t)Hq, (uint64_t)M};
    uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)Hq * D * 2};
    uint32_t box[3] = {64, (uint32_t)G, (uint32_t)(128 / G)};
    TRY(make_tmap(&e->tm_Q, e->Q, 3, dims, strides, box));
  }
  e->ar_buf[0] = reinterpret_cast<float*>(b + a.off_ar);
  e->ar_buf[1] = e->ar_buf[0] + (size_t)M * d;
  e->tp_flags = reinterpret_cast<long long*>(b + a.off_tpflags);
  e->tp_counter = e->tp_flags + 8;
  e->chain_bar = reinterpret_cast<unsigned*>(e->tp_flags + 9);
  e->attn_ctr = reinterpret_cast<unsigned*>(e->tp_flags + 11);
  CK(cudaMemsetAsync(e->tp_flags, 0, 9 * 8 + 16 + 16, st));
  for (int r = 0; r < 8; ++r) {
    e->peer_flags.p[r] = nullptr;
    e->peer_ar[0][r] = e->peer_ar[1][r] = nullptr;
  }
  e->peer_flags.p[e->tp_rank] = e->tp_flags;
  e->peer_ar[0][e->tp_rank] = e->ar_buf[0];
  e->peer_ar[1][e->tp_rank] = e->ar_buf[1];
  CK(cudaMallocHost(&e->plan_host, a.plan_ints * 4));
  CK(cudaMallocHost(&e->host_logits, (size_t)e->lim.max_requests * V * 4));
  CK(cudaMallocHost(&e->host_amax, (size_t)e->lim.max_requests * 4));
  CK(cudaEventCreateWithFlags(&e->plan_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(e->plan_ev, st));
  CK(cudaEventCreate(&e->ev0));
  CK(cudaEventCreate(&e->ev1));
  CK(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&e->side_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&e->k2_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->k2_join, cudaEventDisableTiming));
  e->k2_layer_done.assign(e->cfg.n_layers, nullptr);
  for (auto& ev : e->k2_layer_done) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(prepare_kernels());
  CK(cudaStreamSynchronize(st));
  return PIC_OK;
}

extern "C" pic_status pic_engine_create_tp(const pic_model_config* gcfg, const pic_engine_limits* limits,
                                           int32_t device, void* arena, size_t arena_bytes, void* stream,
                                           int32_t tp_rank, int32_t tp_size, pic_engine** out) {
  TRY(validate_cfg(gcfg, limits));
  TRY(validate_tp(gcfg, tp_rank, tp_size));
  const pic_model_config lc = local_cfg(*gcfg, tp_size);
  const pic_model_config* cfg = &lc;
  TRY(validate_cfg(cfg, limits));
  if (!out) return fail(PIC_E_INVALID_ARG, "NULL out");
  *out = nullptr;
  pic_engine* e = new (std::nothrow) pic_engine();
  if (!e) return fail(PIC_E_OOM, "engine allocation failed");
  e->tp_rank = tp_rank;
  e->tp_size = tp_size;
  e->gcfg = *gcfg;
  e->cfg = *cfg;
  e->lim = *limits;
  e->device = device;
  e->host_only = device < 0;
  e->alloc.reset(limits->num_blocks);
  if (!e->host_only) {
    cudaError_t err = cudaSetDevice(device);
    if (err != cudaSuccess) {
      delete e;
      return fail(PIC_E_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(err));
    }
    pic_status s = init_device(e, arena, arena_bytes, reinterpret_cast<cudaStream_t>(stream));
    if (s != PIC_OK) {
      std::string msg = g_err;
      pic_engine_destroy(e);
      g_err = msg;
      return s;
    }
  } else if (arena) {
    delete e;
    return fail(PIC_E_INVALID_ARG, "host-only engine takes no arena");
  } else {
    const ArenaPlan a = plan_arena(*cfg, *limits);
    e->max_seqs = a.max_seqs;
    e->max_tiles = a.max_tiles;
    e->max_bt = a.max_bt;
    e->max_k2 = a.max_k2;
  }
  *out = e;
  return PIC_OK;
}

extern "C" pic_status pic_engine_create(const pic_model_config* cfg, const pic_engine_limits* limits, int32_t device,
                                        void* arena, size_t arena_bytes, void* stream, pic_engine** out) {
  return pic_engine_create_tp(cfg, limits, device, arena, arena_bytes, stream, 0, 1, out);
}

// CUDA IPC handle of this engine's arena (exchanged by the caller, e.g. torch.distributed all_gather).
extern "C" pic_status pic_tp_ipc_handle(pic_engine* e, void* handle64, uint64_t* offset) {
  if (!e || !handle64 || !offset) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine");
  CUdeviceptr base = 0;
  size_t size = 0;
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  if (!fn || reinterpret_cast<GetRange>(fn)(&base, &size, (CUdeviceptr)e->arena) != CUDA_SUCCESS)
    return fail(PIC_E_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle64, &h, sizeof h);
  *offset = (uint64_t)((CUdeviceptr)e->arena - base);
  return PIC_OK;
}

// Open every peer rank's arena (handles[r], offsets[r] from pic_tp_ipc_handle of rank r) and wire the
// peer pointers of the fused all-reduce.  Same layout on every rank (same config and limits).
extern "C" pic_status pic_tp_connect(pic_engine* e, const void* handles, const uint64_t* offsets) {
  if (!e || !handles || !offsets) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine");
  for (int r = 0; r < e->tp_size; ++r) {
    if (r == e->tp_rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, reinterpret_cast<const char*>(handles) + 64 * r, sizeof h);
    void* base = nullptr;
    const cudaError_t oe = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (oe != cudaSuccess)
      return fail(PIC_E_CUDA, "tp rank %d cannot map rank %d's arena (%s): the fused all-reduce needs CUDA IPC "
                  "and peer access between the ranks' GPUs", e->tp_rank, r, cudaGetErrorString(oe));
    e->ipc_opened.push_back(base);
    // the peer's arena lives on its own GPU: this GPU must reach it with loads/stores (NVLink P2P)
    cudaPointerAttributes pa{};
    CK(cudaPointerGetAttributes(&pa, base));
    if (pa.device != e->device) {
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, e->device, pa.device));
      if (!can)
        return fail(PIC_E_CUDA, "tp rank %d: device %d has no peer access to device %d of rank %d", e->tp_rank,
                    e->device, pa.device, r);
    }
    char* peer = reinterpret_cast<char*>(base) + offsets[r];
    const ptrdiff_t d_ar0 = reinterpret_cast<char*>(e->ar_buf[0]) - e->arena;
    const ptrdiff_t d_ar1 = reinterpret_cast<char*>(e->ar_buf[1]) - e->arena;
    const ptrdiff_t d_fl = reinterpret_cast<char*>(e->tp_flags) - e->arena;
    // the arena base is aligned up to 1 KB inside the caller's buffer: same rule on every rank
    char* pb = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(peer) + 1023) & ~uintptr_t(1023));
    e->peer_ar[0][r] = reinterpret_cast<float*>(pb + d_ar0);
    e->peer_ar[1][r] = reinterpret_cast<float*>(pb + d_ar1);
    e->peer_flags.p[r] = pb + d_fl;
  }
  e->tp_connected = true;
  return PIC_OK;
}

extern "C" void pic_engine_destroy(pic_engine* e) {
  if (!e) return;
  if (!e->host_only) {
    for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);
    if (e->plan_host) cudaFreeHost(e->plan_host);
    if (e->host_logits) cudaFreeHost(e->host_logits);
    if (e->host_amax) cudaFreeHost(e->host_amax);
    if (e->plan_ev) cudaEventDestroy(e->plan_ev);
    if (e->ev0) cudaEventDestroy(e->ev0);
    if (e->ev1) cudaEventDestroy(e->ev1);
    if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
    if (e->side_stream) cudaStreamDestroy(e->side_stream);
    if (e->k2_fork) cudaEventDestroy(e->k2_fork);
    if (e->k2_join) cudaEventDestroy(e->k2_join);
    for (auto ev : e->k2_layer_done)
      if (ev) cudaEventDestroy(ev);
    for (void* p : e->ipc_opened) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t ev : e->ev_pool) cudaEventDestroy(ev);
  }
  delete e;
}

// ============================================================================ planner (a1)
static pic_status assemble(pic_engine* e, const pic_segment* segs, int32_t n_segs, LinkPlanHost& p) {
  if (!segs && n_segs) return fail(PIC_E_INVALID_ARG, "NULL segments");
  if (n_segs <= 0) return fail(PIC_E_EMPTY_INPUT, "empty message list");
  int64_t N = 0;
  for (int i = 0; i < n_segs; ++i) {
    const pic_segment& s = segs[i];
    if (s.kind == PIC_SEG_CACHED) {
      auto it = e->store.find(s.id);
      if (it == e->store.end()) return fail(PIC_E_MISSING_CACHE, "segment %d: unknown or expired cache id %llu", i,
                                            (unsigned long long)s.id);
      N += (int64_t)it->second.tokens.size();
    } else if (s.kind == PIC_SEG_TOKENS) {
      if (s.n_tokens <= 0) return fail(PIC_E_EMPTY_INPUT, "segment %d: empty literal segment", i);
      if (!s.tokens) return fail(PIC_E_INVALID_ARG, "segment %d: NULL tokens", i);
      N += s.n_tokens;
    } else {
      return fail(PIC_E_INVALID_ARG, "segment %d: bad kind %d", i, s.kind);
    }
  }
  if (N > e->lim.max_tokens || N > e->cfg.max_pos)
    return fail(PIC_E_CAPACITY, "linked prompt of %lld tokens exceeds max_tokens %d / max_pos %d", (long long)N,
                e->lim.max_tokens, e->cfg.max_pos);
  p = LinkPlanHost();
  p.N = (int)N;
  p.tok.reserve(N);
  p.src_cid.reserve(N);
  p.src_row.reserve(N);
  p.dynamic.assign(N, 0);
  int32_t pos = 0;
  for (int i = 0; i < n_segs; ++i) {
    const pic_segment& s = segs[i];
    if (s.kind == PIC_SEG_CACHED) {
      const ChunkRec& c = e->store.at(s.id);
      const int n = (int)c.tokens.size();
      p.chunk_id.push_back(s.id);
      p.chunk_start.push_back(pos);
      p.chunk_len.push_back(n);
      p.chunk_delta.push_back(pos - c.c0);  // Δ_c = s_c − c0 (reading R1)
      for (int j = 0; j < n; ++j) {
        p.tok.push_back(c.tokens[j]);
        p.src_cid.push_back((int32_t)(s.id & 0x7FFFFFFF));
        p.src_row.push_back(j);
      }
      pos += n;
    } else {
      for (int j = 0; j < s.n_tokens; ++j) {
        const int32_t t = s.tokens[j];
        if (t < 0 || t >= e->cfg.vocab) return fail(PIC_E_TOKEN, "segment %d token %d = %d out of range", i, j, t);
        p.tok.push_back(t);
        p.src_cid.push_back(-1);
        p.src_row.push_back(-1);
        p.dynamic[pos + j] = 1;
      }
      pos += s.n_tokens;
    }
  }
  return PIC_OK;
}

static pic_status check_params(const pic_link_params* pr) {
  if (!pr) return fail(PIC_E_INVALID_ARG, "NULL params");
  if (pr->alg < PIC_NAIVE || pr->alg > PIC_LEGOLINK0) return fail(PIC_E_INVALID_ARG, "unknown algorithm %d", pr->alg);
  if (pr->alg == PIC_LEGOLINK && pr->k < 0) return fail(PIC_E_INVALID_ARG, "LegoLink k < 0");
  if (pr->alg == PIC_CACHEBLEND && (pr->r_percent < 0 || pr->r_percent > 100))
    return fail(PIC_E_INVALID_ARG, "CacheBlend R outside [0,100]");
  if (pr->alg == PIC_CACHEBLEND && pr->check_layer < 0) return fail(PIC_E_INVALID_ARG, "check_layer < 0");
  return PIC_OK;
}

// Selected set: Naive = dynamic; FR = all; LegoLink(k) = dynamic ∪ first
// min(k, n_c) rows of every chunk not starting at index 0 (R6, R7); CacheBlend = dynamic
// (its cached rows are chosen at the check layer).  Then ∪ {N−1} (R8).
static void select_rows(const pic_link_params* pr, LinkPlanHost& p) {
  std::vector<uint8_t> s(p.N, 0);
  for (int i = 0; i < p.N; ++i) s[i] = p.dynamic[i];
  if (pr->alg == PIC_FULL) std::fill(s.begin(), s.end(), 1);
  if (pr->alg == PIC_LEGOLINK)
    for (size_t c = 0; c < p.chunk_start.size(); ++c) {
      if (p.chunk_start[c] == 0) continue;
      const int k = std::min(pr->k, p.chunk_len[c]);
      for (int j = 0; j < k; ++j) s[p.chunk_start[c] + j] = 1;
    }
  s[p.N - 1] = 1;
  p.sel.clear();
  for (int i = 0; i < p.N; ++i)
    if (s[i]) p.sel.push_back(i);
}

static int32_t slot_of(const std::vector<int32_t>& bt, int32_t i) { return bt[i / 16] * 16 + i % 16; }

// Shared-block link (pic_link_params.kv_share).  Linked block b (rows 16b..16b+15) is
// linked by reference to a chunk-store block iff its 16 rows are all unselected rows of one cached
// chunk c whose start s_c is 16-aligned (so they are exactly store block (16b − s_c)/16 of c); its keys
// then keep their compile positions and carry Δ_c (0 without re-base), applied by the attention when it
// loads them.  Every other block is fresh (a2 copies its unselected cached rows, a5 scatters the rest).
// shared[b] = store block id or -1; delta[b] = Δ to apply (0 for fresh blocks).  Returns #fresh.
// kv_share 2: the same blocks qualify, but only their V is linked by reference (vshared[b] = store block);
// K gets a fresh block that a2 fills with the re-based keys, so the attention reads K without re-basing.
static int plan_blocks(const pic_engine* e, const pic_link_params* pr, const LinkPlanHost& p,
                       std::vector<int32_t>& shared, std::vector<int32_t>& delta, std::vector<int32_t>* vshared = nullptr) {
  const int nb = (p.N + 15) / 16;
  shared.assign(nb, -1);
  delta.assign(nb, 0);
  if (vshared) vshared->assign(nb, -1);
  if (pr->kv_share && pr->alg != PIC_CACHEBLEND) {
    std::vector<uint8_t> in_sel(p.N, 0);
    for (int32_t i : p.sel) in_sel[i] = 1;
    for (size_t c = 0; c < p.chunk_start.size(); ++c) {
      const int s0 = p.chunk_start[c], n = p.chunk_len[c];
      if (s0 % 16) continue;
      const ChunkRec& ch = e->store.at(p.chunk_id[c]);
      for (int j = 0; j + 16 <= n; j += 16) {
        bool clean = true;
        for (int r = 0; r < 16 && clean; ++r) clean = !in_sel[s0 + j + r];
        // kv_share 3: every block inside an aligned chunk keeps the chunk's compile frame (Δ), fresh or not
        if (pr->kv_share == 3) delta[(s0 + j) / 16] = pr->rebase ? p.chunk_delta[c] : 0;
        if (!clean) continue;
        if (pr->kv_share == 2) {
          if (vshared) (*vshared)[(s0 + j) / 16] = ch.blocks[j / 16];
          continue;
        }
        shared[(s0 + j) / 16] = ch.blocks[j / 16];
        delta[(s0 + j) / 16] = pr->rebase ? p.chunk_delta[c] : 0;
      }
    }
  }
  int fresh = 0;
  for (int b = 0; b < nb; ++b) fresh += shared[b] < 0;
  return fresh;
}

// Block table of a link: shared blocks in place, fresh ids (lowest-free-first, in block order) elsewhere.
static std::vector<int32_t> merge_blocks(const std::vector<int32_t>& shared, const std::vector<int32_t>& fresh) {
  std::vector<int32_t> bt(shared.size());
  size_t k = 0;
  for (size_t b = 0; b < shared.size(); ++b) bt[b] = shared[b] >= 0 ? shared[b] : fresh[k++];
  return bt;
}

// LegoLink-0 links only chunks compiled with a dummy prefix (S:324 variant mismatch); its selection is
// Naive's ("skips recomputation entirely").
static pic_status check_variant(const pic_engine* e, const pic_link_params* pr, const LinkPlanHost& p) {
  if (pr->alg != PIC_LEGOLINK0) return PIC_OK;
  for (size_t c = 0; c < p.chunk_id.size(); ++c)
    if (e->store.at(p.chunk_id[c]).c0 <= 0)
      return fail(PIC_E_VARIANT, "legolink0: cache id %llu was compiled without a dummy prefix",
                  (unsigned long long)p.chunk_id[c]);
  return PIC_OK;
}

extern "C" pic_status pic_plan(pic_engine* e, const pic_segment* segs, int32_t n_segs, const pic_link_params* pr,
                               pic_plan_out* out) {
  if (!e || !out) return fail(PIC_E_INVALID_ARG, "NULL engine/out");
  TRY(check_params(pr));
  LinkPlanHost p;
  TRY(assemble(e, segs, n_segs, p));
  TRY(check_variant(e, pr, p));
  select_rows(pr, p);
  const int nb = (p.N + 15) / 16;
  if (out->capacity < p.N) return fail(PIC_E_LAYOUT, "plan capacity %d < N %d", out->capacity, p.N);
  out->n_tokens = p.N;
  out->n_sel = (int)p.sel.size();
  out->n_chunks = (int)p.chunk_start.size();
  out->n_blocks = nb;
  std::vector<int32_t> shared, bdelta;
  const int n_fresh = plan_blocks(e, pr, p, shared, bdelta);
  std::vector<int32_t> fresh = e->alloc.peek(n_fresh);
  if ((int)fresh.size() < n_fresh) return fail(PIC_E_CAPACITY, "pool has %zu free blocks, need %d", fresh.size(), n_fresh);
  const std::vector<int32_t> bt = merge_blocks(shared, fresh);
  out->n_shared = nb - n_fresh;
  if (out->block_delta) std::copy(bdelta.begin(), bdelta.end(), out->block_delta);
  if (out->sel) std::copy(p.sel.begin(), p.sel.end(), out->sel);
  if (out->tok) std::copy(p.tok.begin(), p.tok.end(), out->tok);
  if (out->src)
    for (int i = 0; i < p.N; ++i) {
      out->src[2 * i] = p.src_cid[i];
      out->src[2 * i + 1] = p.src_row[i];
    }
  if (out->chunks)
    for (size_t c = 0; c < p.chunk_start.size(); ++c) {
      out->chunks[3 * c] = p.chunk_start[c];
      out->chunks[3 * c + 1] = p.chunk_len[c];
      out->chunks[3 * c + 2] = p.chunk_delta[c];
    }
  if (out->block_table) std::copy(bt.begin(), bt.end(), out->block_table);
  if (out->slot)
    for (size_t r = 0; r < p.sel.size(); ++r) out->slot[r] = slot_of(bt, p.sel[r]);
  return PIC_OK;
}

// ============================================================================ forward (a2..a10)
struct PlanPack {  // dynamic packing of the plan arrays into one H2D copy
  std::vector<int32_t>* host = nullptr;
  size_t n = 0;
  int32_t* base_dev = nullptr;
  int32_t* put(const std::vector<int32_t>& v, size_t reserve = 0) {
    const size_t off = n;
    const size_t len = std::max(v.size(), reserve);
    n += (len + 31) & ~size_t(31);
    host->resize(n, 0);
    std::copy(v.begin(), v.end(), host->begin() + off);
    return base_dev + off;
  }
};

struct GemmChoice {
  int bn, splits;
  int pair = 0;  // 1: CTA-pair kernel (cta_group::2, 256-row M-tiles)
};

// CTA pairs (cta_group::2) halve the B operand bytes staged and read per SM and FLOP.  Measured
// (scripts/gemm_pair_probe.py): 12-22% faster per unit of work on the cfg4 shapes with zero operands,
// but only 3-5% with random operands — the tensor-bound GEMMs run power-capped (~1.5 GHz), and the
// pair saves operand traffic, not tensor energy — and slower end to end in the engine (cfg4 128 vs
// 118 ms, cfg3 CacheBlend-15 20.4 vs 18.3 ms).  Opt-in (PIC_PAIR=1); the choice then compares
// waves x per-unit cost with pair units at kPairCost.
constexpr double kPairCost = 0.85;
static bool pairs_enabled() {
  static const bool on = getenv("PIC_PAIR") != nullptr;
  return on;
}
// CTA pairs for the fused-epilogue (unsplit) GEMMs: QKV + RoPE/scatter, O / down + residual (+ fused norm).
// Opt-in (PIC_PAIR_FUSED=1): measured neutral at cfg4 (819.7 / 822.2 vs 818.3 / 819.3 ms per step, same box),
// unlike the gate/up GEMM (default pair, 4.9% faster).
static bool fused_pairs() {
  static const bool on = getenv("PIC_PAIR_FUSED") != nullptr;
  return on;
}
static double gemm_cost(int M, int N, int kblk, int bn, int sp, int pair) {
  const int cl = pair ? 2 : 1;
  const long units = (long)((M + 128 * cl - 1) / (128 * cl)) * ((N + bn - 1) / bn) * sp;
  const long slots = 148 / cl;
  const long waves = (units + slots - 1) / slots;
  const int kper = (kblk + sp - 1) / sp;
  return (double)waves * kper * (bn + 32) * (pair ? kPairCost : 1.0) + (sp - 1) * 0.02 * kblk * bn;
}

// Tile / split-K choice (measured, scripts/gemm_sweep.py): a CTA streams ~40 GB/s of weights, so a
// GEMM wants every SM busy in ONE wave.  bn=128 with split-K when its tiles fit in a wave (skinny M:
// QKV 48x3, O and down 32x4 CTAs), otherwise bn=256 (fewer A re-reads, full-rate UMMA N=256).
static GemmChoice choose_gemm(const pic_engine* e, int M, int N, int K) {
  const int kblk = K / 64, mt = (M + 127) / 128;
  const int base_units = mt * ((N + 255) / 256);  // the bn-256 rule below at several m-tiles
  if (mt >= 2 && wave_fit() && base_units <= 132) {
    // (only when that rule would leave SMs idle in a single wave: at several waves bn 256's higher
    // per-instruction efficiency won in measurement, cfg4 124 vs 137 ms)
    // Several m-tiles: the GEMM is MMA-bound, so its time is waves x per-unit work.  Pick the N-tile
    // (and split-K) that quantises best onto 148 SMs, e.g. cfg3's O/down (M = 608, N = 4096): bn 144 ->
    // 145 units in one wave instead of bn 256 -> 80 units on 80 SMs.
    GemmChoice best{256, 1};
    double best_cost = 1e300;
    for (int bn : {256, 224, 208, 192, 176, 160, 144, 128})
      for (int sp = 1; sp <= 4; ++sp) {
        if (sp > 1 && (sp > kblk / 4 || (size_t)sp * M * N > e->ws_floats)) continue;
        const int units = mt * ((N + bn - 1) / bn) * sp;
        const int waves = (units + 147) / 148, kper = (kblk + sp - 1) / sp;
        const double cost = (double)waves * kper * (bn + 32) + (sp - 1) * 0.02 * kblk * bn;  // + partial traffic
        if (cost < best_cost - 1e-9) {
          best_cost = cost;
          best = GemmChoice{bn, sp};
        }
      }
    return best;
  }
  const int t128 = mt * ((N + 127) / 128), t256 = mt * ((N + 255) / 256);
  GemmChoice g = t128 <= 148 ? GemmChoice{128, 148 / t128} : GemmChoice{256, std::max(1, 148 / t256)};
  if (mt == 1 && t128 > 148 && wave_fit()) {
    // one m-tile, too many N-tiles for a wave at bn 128 (the LM head: N = vocab): each CTA streams
    // bn·K weights per unit, so minimise waves x bn (vocab 32000: bn 224 -> 143 units, one wave)
    int best = 256, best_cost = ((N + 255) / 256 + 147) / 148 * 256;
    for (int bn : {224, 208, 192, 176, 160, 144}) {
      const int cost = ((N + bn - 1) / bn + 147) / 148 * bn;
      if (cost < best_cost) {
        best = bn;
        best_cost = cost;
      }
    }
    g = GemmChoice{best, 1};
  }
  g.splits = std::max(1, std::min(g.splits, kblk / 4));
  while (g.splits > 1 && (size_t)g.splits * M * N > e->ws_floats) --g.splits;
  if (mt >= 2 && pairs_enabled()) {
    double best = gemm_cost(M, N, kblk, g.bn, g.splits, 0);
    for (int bn : {256, 224, 192, 128})
      for (int sp = 1; sp <= 4; ++sp) {
        if (!gemm_pair_supported(bn) || (sp > 1 && (sp > kblk / 4 || (size_t)sp * M * N > e->ws_floats))) continue;
        const double c = gemm_cost(M, N, kblk, bn, sp, 1);
        if (c < best - 1e-9) {
          best = c;
          g = GemmChoice{bn, sp, 1};
        }
      }
  }
  return g;
}

// Fused gate/up + SwiGLU GEMM (N-tile fixed at 2g by the weight interleave): CTA pair when it costs less.
// Default on (PIC_NO_PAIR_SWIGLU=1: off): with the convergent MMA issue the pair kernel measured 3% faster
// per cfg4 step for the gate/up GEMM (830 vs 854-859 ms, same box), the largest GEMM of the layer.
static bool swiglu_pair(const pic_engine* e, int M, int N2) {
  static const bool sw = getenv("PIC_NO_PAIR_SWIGLU") == nullptr;
  const int bn = 2 * e->gu_group;
  if (M <= 128 || !(pairs_enabled() || sw) || !gemm_pair_supported(bn) || e->f32) return false;
  return gemm_cost(M, N2, 1, bn, 1, 1) < gemm_cost(M, N2, 1, bn, 1, 0) - 1e-9;
}

// Weight tensor map with a `box`-row box (N-tiles other than 64/128/256, CTA-pair halves), built on
// first use and cached per (matrix, box).
static pic_status weight_map(pic_engine* e, const void* B_ptr, int N, int K, int box, const CUtensorMap** out) {
  const auto key = std::make_pair(B_ptr, box);
  auto it = e->wmaps.find(key);
  if (it == e->wmaps.end()) {
    CUtensorMap m;
    TRY(make_tmap_2d(&m, const_cast<void*>(B_ptr), (uint64_t)N, (uint64_t)K, (uint32_t)box));
    it = e->wmaps.emplace(key, m).first;
  }
  *out = &it->second;
  return PIC_OK;
}

struct Runner {
  pic_engine* e;
  cudaStream_t st;
  int64_t launches = 0;
  pic_status gemm(const CUtensorMap& A, const CUtensorMap* B3, int M, int N, int K, int* splits_out,
                  const void* A_ptr = nullptr, const void* B_ptr = nullptr) {
    if (e->f32) {  // fp32 debug build: CUDA-core GEMM, exact bf16 weight products, fp32 activations
      *splits_out = 1;
      ++launches;
      PROF("gemm", (double)N * K * 2 + (double)M * K * 4 + (double)M * N * 4, 2.0 * M * N * K,
           launch_gemm_simt_f32(reinterpret_cast<const float*>(A_ptr), B_ptr, e->ws, M, N, K, st));
      return PIC_OK;
    }
    GemmChoice g = choose_gemm(e, M, N, K);
    *splits_out = g.splits;
    if (debug_sync()) fprintf(stderr, "[pic] gemm M=%d N=%d K=%d bn=%d splits=%d\n", M, N, K, g.bn, g.splits);
    ++launches;
    const int box = g.pair ? g.bn / 2 : g.bn;  // a CTA pair loads half of the N-tile per CTA
    const CUtensorMap* Bm = (box == 64 || box == 128 || box == 256) ? &B3[bn_index(box)] : nullptr;
    if (!Bm) TRY(weight_map(e, B_ptr, N, K, box, &Bm));
    // algorithmic bytes: the weights, read once per forward; activations and split-K
    // partials are not counted (they are the non-algorithmic part of the measured DRAM traffic)
    PROF("gemm", (double)N * K * 2, 2.0 * M * N * K,
         launch_gemm_partial(A, *Bm, e->ws, M, N, K, g.splits, g.bn, st, 0, GemmNext{}, g.pair));
    return PIC_OK;
  }
  // Unsplit (tensor-bound) choice whose N-tile has a fused-epilogue instance, else nullptr.
  const CUtensorMap* fused_map(const CUtensorMap* B3, const void* B_ptr, int M, int N, int K, bool heads, int* bn,
                               pic_status* err, int* pair = nullptr) {
    *err = PIC_OK;
    if (pair) *pair = 0;
    if (e->f32 || !epi_fuse()) return nullptr;
    GemmChoice g = choose_gemm(e, M, N, K);
    if (g.pair) return nullptr;  // PIC_PAIR's split choice: not a fused shape
    if (g.splits != 1 || !(heads ? (g.bn == 128 || g.bn == 256) : gemm_resid_supported(g.bn))) return nullptr;
    if (pair && fused_pairs() && M > 256) {
      // CTA pair (256-row M-tiles) when its waves x per-unit cost is lower (same N-tile candidates)
      double best = gemm_cost(M, N, K / 64, g.bn, 1, 0);
      for (int b : {256, 224, 192, 128}) {
        if (!gemm_pair_supported(b) || (heads && b != 128 && b != 256)) continue;
        const double c = gemm_cost(M, N, K / 64, b, 1, 1);
        if (c < best - 1e-9) {
          best = c;
          g = GemmChoice{b, 1, 1};
        }
      }
    }
    const int box = g.pair ? g.bn / 2 : g.bn;  // a CTA pair loads half of the N-tile per CTA
    const CUtensorMap* Bm = (box == 64 || box == 128 || box == 256) ? &B3[bn_index(box)] : nullptr;
    if (!Bm) *err = weight_map(e, B_ptr, N, K, box, &Bm);
    *bn = g.bn;
    if (pair) *pair = g.pair;
    return *err == PIC_OK ? Bm : nullptr;
  }
  // a7 / a8-down: h += A·Bᵀ in the epilogue of an unsplit GEMM (*splits_out = 0), else split-K partials
  // for the residual kernel.  Not under tensor parallelism (the partials are all-reduced first).
  // norm_gain (nullable): also write x = bf16(h_new·g) + Σh² partials (*norm_tiles = n-tiles, 0 if not fused)
  pic_status gemm_resid(const CUtensorMap& A, const CUtensorMap* B3, int M, int N, int K, float* h, int* splits_out,
                        const void* A_ptr, const void* B_ptr, const float* norm_gain = nullptr, void* xg = nullptr,
                        int* norm_tiles = nullptr) {
    if (norm_tiles) *norm_tiles = 0;
    int bn = 0, pair = 0;
    pic_status err;
    const CUtensorMap* Bm = e->tp_size == 1 ? fused_map(B3, B_ptr, M, N, K, false, &bn, &err, &pair) : nullptr;
    if (e->tp_size == 1) TRY(err);
    if (!Bm) return gemm(A, B3, M, N, K, splits_out, A_ptr, B_ptr);
    *splits_out = 0;
    ++launches;
    GemmEpi ep{};
    if (norm_gain && (N + bn - 1) / bn <= kSsqStride) {
      ep.norm_gain = norm_gain;
      ep.xg = xg;
      ep.ssq = e->ssq;
      if (norm_tiles) *norm_tiles = (N + bn - 1) / bn;
    }
    PROF("gemm", (double)N * K * 2, 2.0 * M * N * K, launch_gemm_resid(A, *Bm, h, M, N, K, bn, st, GemmNext{}, ep, pair));
    return PIC_OK;
  }
  // will this QKV projection run on the fused-epilogue GEMM (so it can take a fused-norm input)?
  bool qkv_fusable(const LayerW& w, int M) {
    if (e->cfg.head_dim != 128) return false;
    int bn = 0;
    pic_status err;
    const int qkv = (e->cfg.n_heads + 2 * e->cfg.n_kv_heads) * 128;
    return fused_map(w.tm_qkv, w.qkv, M, qkv, e->cfg.d_model, true, &bn, &err) != nullptr && err == PIC_OK;
  }
  // a5: QKV projection with RoPE + scatter in the epilogue of an unsplit GEMM (*fused = true), else
  // split-K partials for qkv_rope_scatter.
  pic_status gemm_qkv(const CUtensorMap& A, const CUtensorMap* B3, int M, int N, int K, const GemmEpi& ep,
                      int* splits_out, bool* fused, const void* A_ptr, const void* B_ptr) {
    int bn = 0, pair = 0;
    pic_status err;
    const CUtensorMap* Bm = e->cfg.head_dim == 128 ? fused_map(B3, B_ptr, M, N, K, true, &bn, &err, &pair) : nullptr;
    if (e->cfg.head_dim == 128) TRY(err);
    *fused = Bm != nullptr;
    if (!Bm) return gemm(A, B3, M, N, K, splits_out, A_ptr, B_ptr);
    *splits_out = 1;
    ++launches;
    PROF("gemm", (double)N * K * 2, 2.0 * M * N * K, launch_gemm_qkv(A, *Bm, ep, M, N, K, bn, st, GemmNext{}, pair));
    return PIC_OK;
  }
};

// Enqueue the whole forward on `st`.  Plan arrays are already on the device at the given pointers.
struct DevPlan {
  int32_t *tok, *pos, *slot, *seq, *tiles, *seq_bt_off, *bt, *bdelta, *k2_src, *k2_dst, *k2_delta, *head_map;
  int32_t *vbt = nullptr, *k2_vcopy = nullptr;  // kv_share 2: V block table, per-a2-row V copy flag
  int32_t* kpos = nullptr;                       // kv_share 3: K heads' RoPE positions (chunk frames)
  int32_t *cb_cand, *cb_forced, *cb_sel2, *cb_pos2, *cb_slot2, *cb_keep, *cb_count, *tiles2, *head_map2;
  int n_tiles, n_tiles2;
  int32_t *attn_work, *attn_nsplit, *attn_work2, *attn_nsplit2;
};

static pic_status enqueue_forward(pic_engine* e, const Fwd& f, const DevPlan& dp, cudaStream_t st, float* debug_hidden,
                                  int64_t* n_launch) {
  const pic_model_config& c = e->cfg;
  const int L = c.n_layers, d = c.d_model, D = c.head_dim, Hq = c.n_heads, Hkv = c.n_kv_heads, F = c.ffn_dim;
  const int qkv = (Hq + 2 * Hkv) * D;
  const float eps = (float)c.rms_eps;
  Runner R{e, st};
  char* Kp = reinterpret_cast<char*>(e->Kpool);
  char* Vp = reinterpret_cast<char*>(e->Vpool);
  const size_t lbytes = (size_t)e->layer_stride * (e->f32 ? 4 : 2);

  // a2: the first K2 layer on the main stream; every later layer as its own launch on a side stream,
  // each recording an event that the main stream waits for just before that layer needs the rows (its
  // attention; CacheBlend: its scatter, see below).  The side stream runs ahead, so the HBM-bound re-base
  // overlaps the tensor-bound projections of the first layers instead of delaying layer k2_layer0+1.
  const bool k2_side = !f.k2_src.empty() && f.k2_layer0 + 1 < L && !e->profiling && k2_overlap() && e->side_stream;
  if (!f.k2_src.empty() && f.k2_layer0 < L) {
    const int n_first = k2_side ? 1 : L - f.k2_layer0;
    ++R.launches;
    PROF("kv_link", 8.0 * D * Hkv * (double)f.k2_src.size() * n_first, 0, launch_kv_link(e->Kpool, e->Vpool, dp.k2_src, dp.k2_dst, dp.k2_delta, (int)f.k2_src.size(), f.k2_layer0,
                      n_first, e->layer_stride, Hkv, D, e->cos_t, e->sin_t, f.rebase, st, e->f32, 148 * 4, dp.k2_vcopy));
    if (k2_side) {
      CK(cudaEventRecord(e->k2_fork, st));
      CK(cudaStreamWaitEvent(e->side_stream, e->k2_fork, 0));
      for (int l = f.k2_layer0 + 1; l < L; ++l) {
        ++R.launches;
        // one CTA per SM: it shares each SM with the persistent GEMM CTA instead of crowding it out
        CKL(launch_kv_link(e->Kpool, e->Vpool, dp.k2_src, dp.k2_dst, dp.k2_delta, (int)f.k2_src.size(), l, 1,
                           e->layer_stride, Hkv, D, e->cos_t, e->sin_t, f.rebase, e->side_stream, e->f32, 148,
                           dp.k2_vcopy));
        CK(cudaEventRecord(e->k2_layer_done[l], e->side_stream));  // joined by layer l (the last by layer L-1)
      }
    }
  }
  ++R.launches;
  PROF("embed", 6.0 * f.M * d, 0, launch_embed(e->E, dp.tok, e->h, f.M, d, st));
  int M = f.M;
  float* hc = e->h;
  const int32_t *pos = dp.pos, *slot = dp.slot, *tiles = dp.tiles;
  int n_tiles = dp.n_tiles;
  const int32_t* head_map = dp.head_map;
  float* prevP = nullptr;
  int prev_s = 0;
  int ar_parity = 0;  // alternates per all-reduce; 2L (link) or 2L-2 (compile) per forward: even
  // residual add (+ RMSNorm): h += Σ partials; under tensor parallelism the partials of every rank are
  // summed straight from peer memory (this rank's splits reduced first, then an epoch barrier)
  auto add_norm = [&](float* Pp, int sp, const float* gain, void* xout, const int32_t* map, int rows,
                      double extra_bytes) -> pic_status {
    if (e->tp_size == 1 || !Pp) {
      PROF("rmsnorm", (double)rows * d * (8 + 4 * (Pp ? sp : 0)) + extra_bytes, 0,
           launch_residual_rmsnorm(hc, Pp, sp, gain, xout, map, rows, d, eps, st, e->f32));
      return PIC_OK;
    }
    float* mine = e->ar_buf[ar_parity];
    PROF("tp_allreduce", (double)rows * d * 4 * (sp + 1), 0, launch_tp_reduce_local(Pp, sp, rows, d, mine, st));
    PROF("tp_allreduce", 0, 0, launch_tp_barrier(e->tp_counter, e->peer_flags, e->tp_rank, e->tp_size, st));
    Srcs srcs{};
    srcs.n = e->tp_size;
    for (int r = 0; r < e->tp_size; ++r) srcs.p[r] = e->peer_ar[ar_parity][r];
    PROF("rmsnorm", (double)rows * d * (8 + 4 * e->tp_size) + extra_bytes, 0,
         launch_residual_rmsnorm_srcs(hc, srcs, gain, xout, map, rows, d, eps, st, e->f32));
    ar_parity ^= 1;
    return PIC_OK;
  };
  auto capture = [&](int layer) -> pic_status {
    if (!debug_hidden) return PIC_OK;
    CK(cudaMemcpyAsync(debug_hidden + (size_t)layer * f.debug_rows * d, hc, (size_t)M * d * 4, cudaMemcpyDeviceToHost,
                       st));
    return PIC_OK;
  };
  // Persistent GEMM chain (gemm_chain.cu) for the weight-streaming regime: one launch per layer runs
  // O-proj, residual+RMSNorm, gate/up+SwiGLU, down, residual+RMSNorm and the next layer's QKV.
  const bool use_chain = chain_enabled() && !e->f32 && e->tp_size == 1 && !f.cb && e->gu_group > 0 && f.M <= 128 &&
                         c.d_model <= 4096 &&
                         f.M > 0;
  bool qkv_done = false;  // this layer's QKV partials were produced by the previous layer's chain
  // fused norm state: x holds bf16(h·g) and e->ssq the row partials of `norm_tiles` n-tiles (0: x is normalised)
  int norm_tiles = 0;
  const bool nf = norm_fuse() && !e->f32 && e->tp_size == 1 && !f.cb && !use_chain;
  auto ep_norm_in = [&](GemmEpi& ep) {
    if (!norm_tiles) return;
    ep.ssq_in = e->ssq;
    ep.ssq_in_n = norm_tiles;
    ep.inv_d = 1.f / (float)d;
    ep.eps = eps;
  };
  bool qkv_fused = false;  // this layer's RoPE + scatter ran in the QKV GEMM's epilogue
  int s_chain_qkv = 0;
  for (int l = 0; l < L; ++l) {
    const LayerW& w = e->layers[l];
    char* Kl = Kp + l * lbytes;
    char* Vl = Vp + l * lbytes;
    int s = 0;
    qkv_fused = false;
    if (qkv_done) {
      s = s_chain_qkv;
      qkv_done = false;
    } else {
      if (!norm_tiles) {
        ++R.launches;
        TRY(add_norm(prevP, prev_s, w.g1, e->x, nullptr, M, (double)M * d * 2));
      }
      if (l > 0) TRY(capture(l - 1));
      if (f.cb && l == f.cb_layer) {  // CacheBlend's check needs the partials of all N rows
        TRY(R.gemm(e->tm_x, w.tm_qkv, M, qkv, d, &s, e->x, w.qkv));
      } else {
        GemmEpi ep{pos, slot, e->cos_t, e->sin_t, e->Q, Kl, Vl, Hq, Hkv};
        ep_norm_in(ep);
        if (pos == dp.pos) ep.kpos = dp.kpos;  // chunk-frame keys (kv_share 3); not CacheBlend's rows
        TRY(R.gemm_qkv(e->tm_x, w.tm_qkv, M, qkv, d, ep, &s, &qkv_fused, e->x, w.qkv));
        if (norm_tiles && !qkv_fused) return fail(PIC_E_CUDA, "internal: fused-norm input reached an unfused QKV GEMM");
      }
      norm_tiles = 0;
    }
    // CacheBlend: the side-stream K2 covers every cached row (the selection is device-side), including
    // the rows this layer's scatter rewrites, so it must land before the scatter, not just before attention
    if (k2_side && f.cb && l > f.k2_layer0) CK(cudaStreamWaitEvent(st, e->k2_layer_done[l], 0));
    if (f.cb && l == f.cb_layer) {
      // a9: CacheBlend selection at the check layer (P:170 steps 3-4)
      if (!f.cb_override) {
        R.launches += 3;
        PROF("cb_select", (double)M * qkv * 4 * s, 0, launch_cb_deviation(e->ws, s, dp.cb_cand, dp.slot, e->cos_t, e->sin_t, Kl, Vl, e->cb_dev, M, Hq, Hkv, D,
                               st, e->f32));
        PROF("cb_select", 4.0 * M, 0, launch_cb_rank(e->cb_dev, dp.cb_keep, M, f.cb_T, st));
        PROF("cb_select", 16.0 * M, 0, launch_cb_compact(dp.cb_keep, dp.cb_forced, dp.bt, dp.cb_sel2, dp.cb_pos2, dp.cb_slot2, dp.cb_count, M,
                             st));
      }
      ++R.launches;
      PROF("cb_select", 8.0 * f.M2 * d, 0, launch_gather_rows(hc, dp.cb_sel2, e->h2, f.M2, d, st));
      hc = e->h2;
      ++R.launches;
      PROF("qkv_rope_scatter", (double)f.M2 * qkv * 4 * s + (double)f.M2 * qkv * 2, 0, launch_qkv_rope_scatter(e->ws, s, M, dp.cb_sel2, dp.cb_pos2, dp.cb_slot2, e->cos_t, e->sin_t, e->Q, Kl, Vl,
                                 f.M2, Hq, Hkv, D, st, e->f32));
      M = f.M2;
      pos = dp.cb_pos2;
      slot = dp.cb_slot2;
      tiles = dp.tiles2;
      n_tiles = dp.n_tiles2;
      head_map = dp.head_map2;
    } else if (!qkv_fused) {
      ++R.launches;
      PROF("qkv_rope_scatter", (double)M * qkv * 4 * s + (double)M * qkv * 2, 0, launch_qkv_rope_scatter(e->ws, s, M, nullptr, pos, slot, e->cos_t, e->sin_t, e->Q, Kl, Vl, M, Hq, Hkv, D,
                                 st, e->f32, pos == dp.pos ? 1 : 0, pos == dp.pos ? dp.kpos : nullptr));
    }
    if (f.compile && l == L - 1) break;  // compile needs only the last layer's K/V
    if (k2_side && !f.cb && l > f.k2_layer0) CK(cudaStreamWaitEvent(st, e->k2_layer_done[l], 0));  // this layer's a2 landed
    // a6 attention — algorithmic work: 4·H_q·D·Σ(p_i+1) FLOPs, K/V of keys 0..max p read once
    double attn_flops = 0, attn_bytes = 0;
    if (e->profiling) {
      const std::vector<int32_t>& pv = (M == f.M) ? f.pos : f.cb_pos2;
      double sp = 0;
      if ((int)pv.size() == M)
        for (int32_t p : pv) sp += p + 1.0;
      else
        sp = (double)M * (f.M / 2.0);  // CacheBlend device-side selection: positions not on the host
      attn_flops = 4.0 * Hq * D * sp;
      for (size_t q = 0; q < f.seq_bt_off.size(); ++q) {
        int mx = 0;
        for (int r = 0; r < (int)f.pos.size(); ++r)
          if (f.seq[r] == (int)q) mx = std::max(mx, f.pos[r] + 1);
        attn_bytes += 2.0 * Hkv * D * 2 * mx;
      }
      attn_bytes += (double)M * Hq * D * 2 * 2;
    }
    if (D == 128 && !e->f32) {
      AttnArgs a{};
      a.work = (tiles == dp.tiles) ? dp.attn_work : dp.attn_work2;
      a.n_work = (tiles == dp.tiles) ? f.attn_n_work : f.attn_n_work2;
      a.tiles = tiles;
      a.seq_bt_off = dp.seq_bt_off;
      a.bt = dp.bt;
      a.row_pos = pos;
      a.M = M;
      a.Hq = Hq;
      a.Hkv = Hkv;
      a.layer = l;
      a.num_blocks = (int)e->lim.num_blocks;
      a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
      a.trace = attn_trace_buffer();
      if (a.trace && !f.attn_pp && (size_t)a.n_work * Hkv > 8192) a.trace = nullptr;  // 32 slots x 8192 CTAs
      a.static_plan = (tiles == dp.tiles) ? 1 : 0;  // CacheBlend's post-selection tiles/positions are device-side
      a.kpool = nullptr;  // L2 prefetch of K/V pages: measured slower (TMA unit busy ahead of the real loads)
      a.vpool = e->Vpool;
      a.bdelta = dp.bdelta;
      a.vbt = dp.vbt;
      a.qrot = f.attn_qrot && tiles == dp.tiles ? 1 : 0;
      if (f.attn_decode && tiles == dp.tiles) a.qrot = f.kv_rot ? 1 : 0;  // decode over chunk frames
      a.cos_t = e->cos_t;
      a.sin_t = e->sin_t;
      a.Q = e->Q;
      g_attn_trace_ctas = !a.trace ? 0 : f.attn_pp ? std::min(a.n_work * Hkv, 148) : a.n_work * Hkv;
      g_attn_trace_pp = f.attn_pp;
      a.o_part = e->o_part;
      a.ml_part = e->ml_part;
      const bool main_tiles = tiles == dp.tiles;
      a.row_nsplit = main_tiles ? dp.attn_nsplit : dp.attn_nsplit2;
      a.O = e->Obuf;  // unsplit q-tiles write their normalised bf16 output here directly
      a.item_ctr = e->attn_ctr;
      static const int attn_debug = getenv("PIC_ATTN_DEBUG") ? atoi(getenv("PIC_ATTN_DEBUG")) : 0;
      a.debug = attn_debug;
      const int max_split = main_tiles ? f.attn_max_split : f.attn_max_split2;
      ++R.launches;
      // chunk-frame links: the persistent Q-side re-base kernel when there are several items per SM (cfg4 wave:
      // 1792 items, attention 178 -> 163 ms per step); with about one item per SM (cfg2, cfg3: split pieces
      // sized for 148 CTAs) the one-CTA-per-item kernel measured faster (cfg2 0.60 vs 0.67 ms, cfg3 2.19 vs
      // 2.31 ms per step).  PIC_NO_ATTN_PERSIST=1 / PIC_ATTN_PERSIST=1 force either kernel (tests, A/B).
      const bool qp = a.qrot && getenv("PIC_NO_ATTN_PERSIST") == nullptr &&
                      ((long)a.n_work * a.Hkv >= 2L * 148 || getenv("PIC_ATTN_PERSIST") != nullptr);
      g_attn_last_kind = (f.attn_decode && main_tiles) ? 5 : qp ? 4 : f.attn_pp ? 2 : a.qrot ? 3 : 1;
      if (f.attn_decode && main_tiles)
        PROF("attention", attn_bytes, attn_flops,
             launch_attention_decode(e->tm_K, e->tm_V, e->tm_K8, e->tm_V8, a, st));
      else if (qp)
        PROF("attention", attn_bytes, attn_flops, launch_attention_qp(e->tm_Q, e->tm_K, e->tm_V, e->tm_K8, e->tm_V8, a, 148, st));
      else if (f.attn_pp)
        PROF("attention", attn_bytes, attn_flops,
             launch_attention_pp(e->tm_Q, e->tm_K, e->tm_V, e->tm_K8, e->tm_V8, a, 148, st));
      else
        PROF("attention", attn_bytes, attn_flops, launch_attention_tc(e->tm_Q, e->tm_K, e->tm_V, e->tm_K8, e->tm_V8, a, st));
      if (max_split > 1) {  // merge the split-KV partials of the split rows only
        ++R.launches;
        PROF("attn_combine", (double)max_split * M * Hq * D * 4 + (double)M * Hq * D * 2, 0,
             launch_attn_combine(e->o_part, e->ml_part, a.row_nsplit, e->Obuf, M, Hq, D, st));
      }
    } else {
      ++R.launches;
      g_attn_last_kind = 6;
      PROF("attention", attn_bytes, attn_flops, launch_attention_simt(e->Q, Kl, Vl, dp.seq, dp.seq_bt_off, dp.bt, pos, e->Obuf, M, Hq, Hkv, D,
                               (float)(1.0 / std::sqrt((double)D)), st, e->f32, dp.bdelta, e->cos_t, e->sin_t, dp.vbt));
    }
    if (use_chain) {
      ChainParams cp{};
      const CUtensorMap* maps[kMaxChainMaps];
      int nm = 0;
      double bytes = 0, flops = 0;
      auto gemm_phase = [&](int type, const CUtensorMap* A, const CUtensorMap* B, int N, int K, void* out,
                            int max_splits = 4) -> int {
        ChainPhase& ph = cp.ph[cp.n_phases++];
        ph.type = type;
        ph.M = M;
        ph.N = N;
        ph.kblk = K / 64;
        ph.bn = type == CHAIN_SWIGLU ? 2 * e->gu_group : 128;
        const int tiles = (N + ph.bn - 1) / ph.bn;
        ph.splits = type == CHAIN_SWIGLU ? 1 : std::max(1, std::min({148 / tiles, ph.kblk / 4, max_splits}));
        while (ph.splits > 1 && (size_t)ph.splits * M * N > e->ws_floats) --ph.splits;
        ph.kper = (ph.kblk + ph.splits - 1) / ph.splits;
        ph.a = nm;
        maps[nm++] = A;
        ph.b = nm;
        maps[nm++] = B;
        ph.out = out;
        bytes += (double)N * K * 2 + (double)M * K * 2 + (double)M * N * (type == CHAIN_SWIGLU ? 1 : 4 * ph.splits);
        flops += 2.0 * M * N * K;
        return ph.splits;
      };
      auto norm_phase = [&](int splits, const float* g) {
        ChainPhase& ph = cp.ph[cp.n_phases++];
        ph.type = CHAIN_NORM;
        ph.M = M;
        ph.N = d;
        ph.bn = 128;
        ph.splits = splits;
        ph.P = e->ws;
        ph.g = g;
        ph.h = hc;
        ph.out = e->x;
        ph.eps = eps;
        bytes += (double)M * d * (8 + 4 * splits + 2);
      };
      const int s_o = gemm_phase(CHAIN_GEMM, &e->tm_O, &w.tm_o[bn_index(128)], d, Hq * D, e->ws);
      norm_phase(s_o, w.g2);
      gemm_phase(CHAIN_SWIGLU, &e->tm_x, &w.tm_gu_fused, 2 * F, d, e->u);
      const int s_dn = gemm_phase(CHAIN_GEMM, &e->tm_u, &w.tm_down[bn_index(128)], d, F, e->ws);
      const bool next = l + 1 < L;
      if (next) {
        const LayerW& wn = e->layers[l + 1];
        norm_phase(s_dn, wn.g1);
        s_chain_qkv = gemm_phase(CHAIN_GEMM, &e->tm_x, &wn.tm_qkv[bn_index(128)], qkv, d, e->ws, 32);
        qkv_done = true;
      }
      cp.bar = e->chain_bar;
      cp.trace = chain_trace_buffer() ? chain_trace_buffer() + (size_t)l * 16 * 148 : nullptr;
      ++R.launches;
      PROF("gemm", bytes, flops, launch_gemm_chain(maps, nm, cp, st));
      if (next) {
        TRY(capture(l));  // h after layer l (written by the chain's second norm phase)
      } else {
        prevP = e->ws;
        prev_s = s_dn;
      }
      continue;
    }
    // a7 O projection, residual + a8 MLP
    const bool gu_pair = e->gu_group > 0 && swiglu_pair(e, M, 2 * F);
    const bool fuse_g2 = nf && e->gu_group > 0;
    TRY(R.gemm_resid(e->tm_O, w.tm_o, M, d, Hq * D, hc, &s, e->Obuf, w.o, fuse_g2 ? w.g2 : nullptr, e->x,
                     &norm_tiles));
    if (!norm_tiles) {
      ++R.launches;
      TRY(add_norm(s ? e->ws : nullptr, s, w.g2, e->x, nullptr, M, (double)M * d * 2));
    }
    if (e->gu_group > 0) {
      ++R.launches;
      const CUtensorMap* Bg = &w.tm_gu_fused;
      if (gu_pair) TRY(weight_map(e, w.gu, 2 * F, d, e->gu_group, &Bg));  // each CTA: the gate or the up half
      GemmEpi ep{};
      ep_norm_in(ep);
      norm_tiles = 0;
      PROF("gemm", (double)2 * F * d * 2, 2.0 * M * 2 * F * d,
           launch_gemm_swiglu(e->tm_x, *Bg, e->u, M, 2 * F, d, 2 * e->gu_group, st, 0, GemmNext{}, gu_pair ? 1 : 0, ep));
    } else {
      TRY(R.gemm(e->tm_x, w.tm_gu, M, 2 * F, d, &s, e->x, w.gu));
      ++R.launches;
      PROF("swiglu", (double)M * 2 * F * 4 * s + (double)M * F * 2, 0, launch_swiglu(e->ws, s, e->u, M, F, st, e->f32));
    }
    // the next layer's a4 fused into this epilogue when its QKV GEMM takes the fused input
    const bool fuse_g1 = nf && l + 1 < L && R.qkv_fusable(e->layers[l + 1], M);
    TRY(R.gemm_resid(e->tm_u, w.tm_down, M, d, F, hc, &s, e->u, w.down, fuse_g1 ? e->layers[l + 1].g1 : nullptr,
                     e->x, &norm_tiles));
    prevP = s ? e->ws : nullptr;
    prev_s = s;
  }
  if (!f.compile) {
    // a10: final norm of the last rows, LM head, argmax
    ++R.launches;
    TRY(add_norm(prevP, prev_s, e->gf, e->x_last, head_map, M, (double)f.n_head * d * 2));
    TRY(capture(L - 1));
    int s = 0;
    TRY(R.gemm(e->tm_xlast, e->tm_lm, f.n_head, c.vocab, d, &s, e->x_last, e->Wlm));
    ++R.launches;
    PROF("logits_argmax", (double)f.n_head * c.vocab * 4 * (s + 1), 0, launch_logits_argmax(e->ws, s, e->logits, e->amax, f.n_head, c.vocab, st));
  }
  *n_launch = R.launches;
  return PIC_OK;
}

static void add_sig(std::vector<int64_t>& sig, const Fwd& f, const DevPlan& dp) {
  sig = {f.M,  dp.n_tiles, (int64_t)f.seq_bt_off.size(), (int64_t)f.bt.size(), (int64_t)f.k2_src.size(), f.k2_layer0,
         f.n_head, f.compile, f.rebase, f.cb, f.cb_layer, f.cb_T, f.M2, f.cb_override, dp.n_tiles2, f.attn_n_work,
         f.attn_n_work2, f.kv_rot, f.attn_pp, f.has_vbt, f.k2_konly, f.has_kpos, f.attn_qrot, f.attn_decode};
  // attention split choice depends on the per-sequence block-table lengths
  for (size_t q = 0; q < f.seq_bt_off.size(); ++q) sig.push_back(f.seq_bt_off[q]);
}

// Balanced split-KV schedules for the attention of this forward (host-known positions; CacheBlend's
// post-check rows use the request length as the causal extent and the kernel clamps).
static void schedule_attention(pic_engine* e, Fwd& f) {
  const int Hkv = e->cfg.n_kv_heads;
  auto build = [&](const std::vector<int32_t>& tiles, const std::vector<int32_t>* pos, int M, int fallback_len,
                   std::vector<int32_t>& work, std::vector<int32_t>& nsplit, int& n_work, int& max_split) {
    const int nt = (int)tiles.size() / 3;
    std::vector<int> n_kv(nt);
    for (int t = 0; t < nt; ++t) {
      int mx = fallback_len - 1;
      if (pos) {
        mx = 0;
        for (int r = 0; r < tiles[3 * t + 2]; ++r) mx = std::max(mx, (*pos)[tiles[3 * t + 1] + r]);
      }
      n_kv[t] = mx / 128 + 1;
    }
    int cap = std::max(1, std::min(32, e->attn_rows_cap / std::max(M, 1)));
    // decode kernel: HBM-bound, so with at least one (sequence, kv-head) item per SM the pieces need no split
    // (cfg4 batch 32: 256 items; 6.22 vs 6.04 TB/s and no combine launch, TPOT -0.2 ms); PIC_DEC_SPLIT=1: A/B
    if (f.attn_decode && (long)nt * Hkv >= 148 && !getenv("PIC_DEC_SPLIT")) cap = 1;
    long total = 0;
    for (int v : n_kv) total += v;
    work.assign(4 * (size_t)(total + nt), 0);
    nsplit.assign(M, 1);
    if (f.attn_pp) {
      max_split = attn_schedule_pp(tiles.data(), nt, n_kv.data(), Hkv, 148, cap, work, nsplit.data());
      n_work = (int)work.size() / 8;
      return;
    }
    max_split = attn_schedule(tiles.data(), nt, n_kv.data(), Hkv, 148, cap, work.data(), &n_work, nsplit.data());
    work.resize(4 * (size_t)n_work);
  };
  // Kernel choice (D = 128, bf16): the ping-pong kernel needs enough tile work to keep 148 persistent
  // CTAs busy with paired lanes (cfg4 wave: 53 k KV-tile iterations, 1.25x faster; cfg2: 544, slower than
  // the one-lane kernel's finer split-KV); shared-block links (K tiles re-based in smem) stay on the
  // one-lane kernel, whose four rotation warps keep up where the ping-pong kernel's two do not (cfg4:
  // 310 vs 200 ms per step).  pic_test_set_attention_kernel(1|2) forces one (tests and A/B only).
  // kv_share 3 links whose every 128-key tile carries one block delta: Q-side re-base in the one-lane kernel
  f.attn_qrot = false;
  if (f.kv_rot && f.qrot_ok && !e->f32 && e->cfg.head_dim == 128 && !getenv("PIC_NO_QROT")) {
    bool uniform = true;
    for (size_t q = 0; q < f.seq_bt_off.size() && uniform; ++q) {
      const size_t b0 = f.seq_bt_off[q], b1 = q + 1 < f.seq_bt_off.size() ? f.seq_bt_off[q + 1] : f.bt.size();
      for (size_t b = b0; b < b1 && uniform; ++b) uniform = f.bdelta[b] == f.bdelta[b0 + (b - b0) / 8 * 8];
    }
    f.attn_qrot = uniform;
  }
  static const bool pp_rot = getenv("PIC_ATTN_PP_ROT") != nullptr;  // A/B: ping-pong also for shared-block links
  bool pp = attn_pp_enabled() && e->cfg.head_dim == 128 && !e->f32 && (!f.kv_rot || pp_rot);
  if (pp) {
    long work = 0;
    for (size_t t = 0; t + 2 < f.tiles.size(); t += 3) {
      int mx = 0;
      for (int r = 0; r < f.tiles[t + 2]; ++r) mx = std::max(mx, f.pos[f.tiles[t + 1] + r]);
      work += mx / 128 + 1;
    }
    pp = work * Hkv >= 148L * 16;
  }
  if (g_attn_force) pp = g_attn_force == 2 && e->cfg.head_dim == 128 && !e->f32;
  if (f.attn_qrot) pp = false;  // the Q-side re-base lives in the one-lane kernel
  // decode (f1): the transposed split-KV kernel, unless keys still need a re-base on load (shared blocks
  // not materialized: the one-lane kernel's K-tile rotation) or PIC_NO_ATTN_DECODE (A/B)
  const bool no_dec = getenv("PIC_NO_ATTN_DECODE") != nullptr;  // read per call (tests toggle it)
  // a cache that still re-bases keys on load qualifies when every 128-key tile carries one Δ (chunk-frame
  // links, kv_share 3): the decode kernel then rotates the query by −Δ per frame
  bool dec_frames = !f.kv_rot;
  if (f.decode && f.kv_rot) {
    dec_frames = true;
    for (size_t q = 0; q < f.seq_bt_off.size() && dec_frames; ++q) {
      const size_t b0 = f.seq_bt_off[q], b1 = q + 1 < f.seq_bt_off.size() ? f.seq_bt_off[q + 1] : f.bt.size();
      for (size_t b = b0; b < b1 && dec_frames; ++b) dec_frames = f.bdelta[b] == f.bdelta[b0 + (b - b0) / 8 * 8];
    }
  }
  f.attn_decode = f.decode && dec_frames && !no_dec && e->cfg.head_dim == 128 && !e->f32 &&
                  attention_decode_supported(e->cfg.n_heads / Hkv);
  if (f.attn_decode) pp = false;
  f.attn_pp = pp;
  build(f.tiles, &f.pos, f.M, 0, f.attn_work, f.attn_nsplit, f.attn_n_work, f.attn_max_split);
  if (f.cb) {
    const int N = f.M;  // single request, all rows at layer 0
    build(f.tiles2, nullptr, f.M2, N, f.attn_work2, f.attn_nsplit2, f.attn_n_work2, f.attn_max_split2);
  }
}

static pic_status run_forward(pic_engine* e, const Fwd& f, cudaStream_t st, bool use_graph, float* debug_hidden) {
  const int Mcap = e->lim.max_rows;
  if (f.M > Mcap) return fail(PIC_E_CAPACITY, "%d rows exceed max_rows %d", f.M, Mcap);
  if ((int)f.tiles.size() / 3 > e->max_tiles || (int)f.seq_bt_off.size() > e->max_seqs ||
      (int)f.bt.size() > e->max_bt || (int)f.k2_src.size() > e->max_k2)
    return fail(PIC_E_CAPACITY, "plan exceeds engine capacities");
  // pack plan arrays
  std::vector<int32_t> host;
  host.reserve(4096);
  PlanPack pk{&host, 0, e->plan_dev};
  DevPlan dp{};
  dp.tok = pk.put(f.tok);
  dp.pos = pk.put(f.pos);
  dp.slot = pk.put(f.slot);
  dp.seq = pk.put(f.seq);
  dp.tiles = pk.put(f.tiles);
  dp.seq_bt_off = pk.put(f.seq_bt_off);
  dp.bt = pk.put(f.bt);
  dp.bdelta = f.kv_rot ? pk.put(f.bdelta) : nullptr;
  dp.vbt = f.has_vbt ? pk.put(f.vbt) : nullptr;
  dp.kpos = f.has_kpos ? pk.put(f.kpos) : nullptr;
  dp.k2_vcopy = f.k2_konly ? pk.put(f.k2_vcopy) : nullptr;
  dp.k2_src = pk.put(f.k2_src);
  dp.k2_dst = pk.put(f.k2_dst);
  dp.k2_delta = pk.put(f.k2_delta);
  dp.head_map = pk.put(f.head_map);
  dp.attn_work = pk.put(f.attn_work);
  dp.attn_nsplit = pk.put(f.attn_nsplit);
  dp.n_tiles = (int)f.tiles.size() / 3;
  if (f.cb) {
    dp.cb_cand = pk.put(f.cb_cand);
    dp.cb_forced = pk.put(f.cb_forced);
    dp.cb_sel2 = pk.put(f.cb_sel2, f.M);
    dp.cb_pos2 = pk.put(f.cb_pos2, f.M);
    dp.cb_slot2 = pk.put(f.cb_slot2, f.M);
    dp.cb_keep = pk.put({}, f.M);
    dp.cb_count = pk.put({}, 1);
    dp.tiles2 = pk.put(f.tiles2);
    dp.head_map2 = pk.put(f.head_map2);
    dp.n_tiles2 = (int)f.tiles2.size() / 3;
    dp.attn_work2 = pk.put(f.attn_work2);
    dp.attn_nsplit2 = pk.put(f.attn_nsplit2);
    e->last_cb_sel2 = dp.cb_sel2;
  }
  if (pk.n > e->plan_cap_ints) return fail(PIC_E_CAPACITY, "plan of %zu ints exceeds %zu", pk.n, e->plan_cap_ints);
  // the previous call's H2D copy must have consumed the pinned staging buffer
  CK(cudaEventSynchronize(e->plan_ev));
  std::memcpy(e->plan_host, host.data(), pk.n * 4);
  CK(cudaMemcpyAsync(e->plan_dev, e->plan_host, pk.n * 4, cudaMemcpyHostToDevice, st));
  CK(cudaEventRecord(e->plan_ev, st));
  e->h2d_last = (int64_t)pk.n * 4;

  int64_t nl = 0;
  if (!use_graph || debug_hidden || debug_sync() || e->profiling) {
    TRY(enqueue_forward(e, f, dp, st, debug_hidden, &nl));
    e->kernels_last = nl;
    return PIC_OK;
  }
  (void)chain_trace_buffer();  // bench-only trace buffers are allocated outside any capture
  (void)attn_trace_buffer();
  std::vector<int64_t> sig;
  add_sig(sig, f, dp);
  auto it = e->graphs.find(sig);
  if (it == e->graphs.end()) {
    // capture on the engine's own stream (the caller's may be the legacy default stream, which
    // cannot be captured); the instantiated graph is then launched on the caller's stream
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
    pic_status s = enqueue_forward(e, f, dp, e->cap_stream, nullptr, &nl);
    cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &g);
    if (s != PIC_OK) {
      if (g) cudaGraphDestroy(g);
      return s;
    }
    if (ce != cudaSuccess) return fail(PIC_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    cudaGraphExec_t ex = nullptr;
    ce = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(PIC_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    if (e->graphs.size() > 64) {
      cudaGraphExecDestroy(e->graphs.begin()->second);
      e->graphs.erase(e->graphs.begin());
    }
    it = e->graphs.emplace(sig, ex).first;
    e->kernels_last = nl;
  }
  CK(cudaGraphLaunch(it->second, st));
  return PIC_OK;
}

// Build the tiles of `rows` rows of sequence `seq` starting at row index r0 of the forward.
static void add_tiles(std::vector<int32_t>& tiles, int seq, int r0, int rows, int qpt) {
  for (int a = 0; a < rows; a += qpt) {
    tiles.push_back(seq);
    tiles.push_back(r0 + a);
    tiles.push_back(std::min(qpt, rows - a));
  }
}

static int qpt_of(const pic_model_config& c) { return 128 / (c.n_heads / c.n_kv_heads); }

// ============================================================================ compile (a0)
// Compile (a0).  m > 0: LegoLink-0 compile (reading R21) — each chunk is prefilled as
// dummy^m ‖ chunk in scratch blocks, then rows m..m+n−1 of every layer are copied into the chunk's
// own blocks (the dummy rows are discarded) and the chunk records c0 = m.
static pic_status compile_impl(pic_engine* e, const int32_t* const* chunks, const int32_t* lens, int32_t n, int32_t m,
                               int32_t dummy_tok, void* stream, pic_cache_id* out_ids, int32_t* err_index) {
  if (err_index) *err_index = -1;
  if (!e || !out_ids || (n > 0 && (!chunks || !lens))) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (n <= 0) return fail(PIC_E_EMPTY_INPUT, "no chunks");
  if (m < 0) return fail(PIC_E_INVALID_ARG, "negative dummy prefix");
  if (dummy_tok < 0) dummy_tok = e->cfg.bos_id;
  if (m > 0 && dummy_tok >= e->cfg.vocab) return fail(PIC_E_TOKEN, "dummy token %d out of range", dummy_tok);
  int64_t need = 0;
  for (int i = 0; i < n; ++i) {
    if (lens[i] <= 0) {
      if (err_index) *err_index = i;
      return fail(PIC_E_EMPTY_INPUT, "chunk %d is empty", i);
    }
    if (!chunks[i]) {
      if (err_index) *err_index = i;
      return fail(PIC_E_INVALID_ARG, "chunk %d is NULL", i);
    }
    if (lens[i] + m > e->cfg.max_pos || lens[i] + m > e->lim.max_tokens) {
      if (err_index) *err_index = i;
      return fail(PIC_E_CAPACITY, "chunk %d of %d (+%d dummy) tokens exceeds max_tokens/max_pos", i, lens[i], m);
    }
    for (int j = 0; j < lens[i]; ++j)
      if (chunks[i][j] < 0 || chunks[i][j] >= e->cfg.vocab) {
        if (err_index) *err_index = i;
        return fail(PIC_E_TOKEN, "chunk %d token %d = %d out of range", i, j, chunks[i][j]);
      }
    need += (lens[i] + 15) / 16 + (m > 0 ? (lens[i] + m + 15) / 16 : 0);
  }
  if (!e->alloc.can(need)) return fail(PIC_E_CAPACITY, "pool has %zu free blocks, compile needs %lld",
                                       e->alloc.free_ids.size(), (long long)need);
  // allocate blocks lowest-free-first in chunk order (then the dummy-prefix scratch blocks)
  std::vector<std::vector<int32_t>> blocks(n), scratch(n);
  for (int i = 0; i < n; ++i) blocks[i] = e->alloc.alloc((lens[i] + 15) / 16);
  if (m > 0)
    for (int i = 0; i < n; ++i) scratch[i] = e->alloc.alloc((lens[i] + m + 15) / 16);
  auto release_scratch = [&]() {
    for (auto& b : scratch) e->alloc.release(b);
  };
  auto rollback = [&]() {
    for (auto& b : blocks) e->alloc.release(b);
    release_scratch();
  };
  if (!e->host_only && e->tp_size > 1 && !e->tp_connected) {
    rollback();
    return fail(PIC_E_INVALID_ARG, "tensor-parallel engine: call pic_tp_connect first");
  }
  if (!e->host_only) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // pack (chunk, row range) pieces into forwards of <= max_rows rows / max_seqs sequences
    const int qpt = qpt_of(e->cfg);
    Fwd f;
    f.compile = true;
    auto flush = [&]() -> pic_status {
      if (f.M == 0) return PIC_OK;
      schedule_attention(e, f);
      pic_status s = run_forward(e, f, st, false, nullptr);
      f = Fwd();
      f.compile = true;
      return s;
    };
    for (int i = 0; i < n; ++i) {
      const std::vector<int32_t>& fb = m > 0 ? scratch[i] : blocks[i];
      const int len = lens[i] + m;
      for (int a = 0; a < len;) {
        const int room = e->lim.max_rows - f.M;
        if (room <= 0 || (int)f.seq_bt_off.size() >= e->max_seqs || (int)f.bt.size() + (int)fb.size() > e->max_bt) {
          pic_status s = flush();
          if (s != PIC_OK) {
            rollback();
            return s;
          }
          continue;
        }
        const int take = std::min(room, len - a);
        const int seq = (int)f.seq_bt_off.size();
        f.seq_bt_off.push_back((int)f.bt.size());
        f.bt.insert(f.bt.end(), fb.begin(), fb.end());
        add_tiles(f.tiles, seq, f.M, take, qpt);
        for (int j = a; j < a + take; ++j) {
          f.tok.push_back(j < m ? dummy_tok : chunks[i][j - m]);
          f.pos.push_back(j);                          // positions from zero
          f.slot.push_back(slot_of(fb, j));
          f.seq.push_back(seq);
        }
        f.M += take;
        a += take;
      }
    }
    pic_status s = flush();
    if (s == PIC_OK && m > 0) {
      // keep rows m..m+n−1 of every layer: the gather of a2 with Δ = 0 (no rotation)
      std::vector<int32_t> src, dst, zero;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < lens[i]; ++j) {
          src.push_back(slot_of(scratch[i], m + j));
          dst.push_back(slot_of(blocks[i], j));
        }
      zero.assign(src.size(), 0);
      std::vector<int32_t> host;
      PlanPack pk{&host, 0, e->plan_dev};
      const int32_t* d_src = pk.put(src);
      const int32_t* d_dst = pk.put(dst);
      const int32_t* d_zero = pk.put(zero);
      if (pk.n > e->plan_cap_ints) {
        s = fail(PIC_E_CAPACITY, "dummy-prefix copy list of %zu ints exceeds %zu", pk.n, e->plan_cap_ints);
      } else {
        cudaError_t ce = cudaEventSynchronize(e->plan_ev);
        if (ce == cudaSuccess) {
          std::memcpy(e->plan_host, host.data(), pk.n * 4);
          ce = cudaMemcpyAsync(e->plan_dev, e->plan_host, pk.n * 4, cudaMemcpyHostToDevice, st);
        }
        if (ce == cudaSuccess) ce = cudaEventRecord(e->plan_ev, st);
        if (ce == cudaSuccess)
          ce = launch_kv_link(e->Kpool, e->Vpool, d_src, d_dst, d_zero, (int)src.size(), 0, e->cfg.n_layers,
                              e->layer_stride, e->cfg.n_kv_heads, e->cfg.head_dim, e->cos_t, e->sin_t, 0, st, e->f32);
        if (ce != cudaSuccess) s = fail(PIC_E_CUDA, "dummy-prefix copy: %s", cudaGetErrorString(ce));
      }
    }
    if (s != PIC_OK) {
      rollback();
      return s;
    }
    cudaError_t ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) {
      rollback();
      return fail(PIC_E_CUDA, "compile: %s", cudaGetErrorString(ce));
    }
  }
  release_scratch();
  for (int i = 0; i < n; ++i) {
    ChunkRec rec;
    rec.tokens.assign(chunks[i], chunks[i] + lens[i]);
    rec.blocks = blocks[i];
    rec.c0 = m;
    const pic_cache_id id = e->next_id++;
    e->store.emplace(id, std::move(rec));
    out_ids[i] = id;
  }
  return PIC_OK;
}

extern "C" pic_status pic_generate_context_cache(pic_engine* e, const int32_t* const* chunks, const int32_t* lens,
                                                 int32_t n, void* stream, pic_cache_id* out_ids, int32_t* err_index) {
  return compile_impl(e, chunks, lens, n, 0, -1, stream, out_ids, err_index);
}

extern "C" pic_status pic_generate_context_cache_ex(pic_engine* e, const int32_t* const* chunks, const int32_t* lens,
                                                    int32_t n, const pic_compile_options* opts, void* stream,
                                                    pic_cache_id* out_ids, int32_t* err_index) {
  return compile_impl(e, chunks, lens, n, opts ? opts->dummy_prefix : 0, opts ? opts->dummy_token : -1, stream,
                      out_ids, err_index);
}

// ============================================================================ link
struct ReqBuild {
  LinkPlanHost p;
  std::vector<int32_t> bt;
  std::vector<int32_t> shared, bdelta;  // f3: per block, store block linked by reference (or -1) and its Δ
  std::vector<int32_t> vshared;         // kv_share 2: per block, store block holding its V (or -1)
  int n_fresh = 0;
};

// Append one request's rows / tiles / K2 work to a forward.
static void append_request(pic_engine* e, const pic_link_params* pr, ReqBuild& rb, int req, Fwd& f) {
  const LinkPlanHost& p = rb.p;
  const int qpt = qpt_of(e->cfg);
  const int seq = (int)f.seq_bt_off.size();
  f.seq_bt_off.push_back((int)f.bt.size());
  f.bt.insert(f.bt.end(), rb.bt.begin(), rb.bt.end());
  f.bdelta.insert(f.bdelta.end(), rb.bdelta.begin(), rb.bdelta.end());
  for (int32_t dl : rb.bdelta) f.kv_rot |= dl != 0;
  for (size_t b = 0; b < rb.bt.size(); ++b) {
    const bool vs = b < rb.vshared.size() && rb.vshared[b] >= 0;
    f.vbt.push_back(vs ? rb.vshared[b] : rb.bt[b]);
    f.has_vbt |= vs;
  }
  const bool cb = pr->alg == PIC_CACHEBLEND;
  const std::vector<int32_t>* rows = &p.sel;
  std::vector<int32_t> all;
  if (cb) {
    all.resize(p.N);
    for (int i = 0; i < p.N; ++i) all[i] = i;
    rows = &all;
  }
  const int r0 = f.M;
  add_tiles(f.tiles, seq, r0, (int)rows->size(), qpt);
  const bool frames = pr->kv_share == 3 && !cb;  // chunk-frame blocks: K stored at compile positions
  f.qrot_ok = frames;
  for (int32_t i : *rows) {
    f.tok.push_back(p.tok[i]);
    f.pos.push_back(i);  // p_i = i (R18)
    const int32_t fr = frames ? rb.bdelta[i / 16] : 0;
    f.kpos.push_back(i - fr);
    f.has_kpos |= fr != 0;
    f.slot.push_back(slot_of(rb.bt, i));
    f.seq.push_back(seq);
    f.head_map.push_back(-1);
  }
  f.M += (int)rows->size();
  f.head_map[f.M - 1] = req;  // last row N−1 (always selected, R8)
  // a2 work list: cached rows not recomputed (CacheBlend: all cached rows, from the check layer on)
  std::vector<uint8_t> in_sel(p.N, 0);
  if (!cb)
    for (int32_t i : p.sel) in_sel[i] = 1;
  for (size_t c = 0; c < p.chunk_start.size(); ++c) {
    const ChunkRec& ch = e->store.at(p.chunk_id[c]);
    for (int j = 0; j < p.chunk_len[c]; ++j) {
      const int i = p.chunk_start[c] + j;
      if (in_sel[i] || rb.shared[i / 16] >= 0) continue;  // recomputed, or linked by reference (f3)
      f.k2_src.push_back(slot_of(ch.blocks, j));
      f.k2_dst.push_back(slot_of(rb.bt, i));
      // a chunk-frame block (kv_share 3) keeps the copied keys at their compile positions
      f.k2_delta.push_back(frames && rb.bdelta[i / 16] != 0 ? 0 : p.chunk_delta[c]);
      const bool vref = !rb.vshared.empty() && rb.vshared[i / 16] >= 0;  // kv_share 2: V stays in the store
      f.k2_vcopy.push_back(vref ? 0 : 1);
      f.k2_konly |= vref;
    }
  }
}

static pic_status link_impl(pic_engine* e, int32_t n_req, const pic_segment* const* segs, const int32_t* n_segs,
                            const pic_link_params* pr, void* stream, pic_linked** out_linked,
                            pic_link_result* results) {
  if (!e || !segs || !n_segs || !results) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (n_req <= 0) return fail(PIC_E_EMPTY_INPUT, "no requests");
  if (n_req > e->lim.max_requests) return fail(PIC_E_CAPACITY, "%d requests exceed max_requests", n_req);
  TRY(check_params(pr));
  const bool cb = pr->alg == PIC_CACHEBLEND;
  if (cb && n_req != 1) return fail(PIC_E_VARIANT, "CacheBlend is single-request");
  if (pr->sel_override && !cb) return fail(PIC_E_VARIANT, "sel_override is a CacheBlend hook");
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine cannot link");
  if (e->tp_size > 1 && !e->tp_connected) return fail(PIC_E_INVALID_ARG, "tensor-parallel engine: call pic_tp_connect first");
  if (e->tp_size > 1 && cb) return fail(PIC_E_VARIANT, "CacheBlend is not supported with tensor parallelism");
  std::vector<ReqBuild> reqs(n_req);
  int64_t need = 0;
  for (int r = 0; r < n_req; ++r) {
    TRY(assemble(e, segs[r], n_segs[r], reqs[r].p));
    TRY(check_variant(e, pr, reqs[r].p));
    select_rows(pr, reqs[r].p);
    reqs[r].n_fresh = plan_blocks(e, pr, reqs[r].p, reqs[r].shared, reqs[r].bdelta, &reqs[r].vshared);
    need += reqs[r].n_fresh;
  }
  if (!e->alloc.can(need)) return fail(PIC_E_CAPACITY, "pool has %zu free blocks, link needs %lld",
                                       e->alloc.free_ids.size(), (long long)need);
  Fwd f;
  f.rebase = pr->rebase;
  f.n_head = n_req;
  for (int r = 0; r < n_req; ++r) {
    reqs[r].bt = merge_blocks(reqs[r].shared, e->alloc.alloc(reqs[r].n_fresh));
    for (int32_t b : reqs[r].shared)
      if (b >= 0) e->alloc.retain(b);  // the linked cache holds the chunk-store block too
    for (int32_t b : reqs[r].vshared)
      if (b >= 0) e->alloc.retain(b);  // kv_share 2: the store block holding this block's V
  }
  auto rollback = [&]() {
    for (auto& rb : reqs) {
      e->alloc.release(rb.bt);
      for (int32_t b : rb.vshared)
        if (b >= 0) e->alloc.release({b});
    }
  };
  for (int r = 0; r < n_req; ++r) append_request(e, pr, reqs[r], r, f);
  f.debug_rows = std::max(reqs[0].p.N, f.M);  // debug_hidden row stride (pic.h)
  if (cb) {
    const LinkPlanHost& p = reqs[0].p;
    const int N = p.N;
    f.cb = pr->check_layer < e->cfg.n_layers;
    f.cb_layer = pr->check_layer;
    f.k2_layer0 = std::min(pr->check_layer, e->cfg.n_layers);
    int n_cached = 0;
    f.cb_cand.assign(N, 0);
    f.cb_forced.assign(N, 0);
    for (int i = 0; i < N; ++i) {
      if (!p.dynamic[i]) ++n_cached;
      f.cb_cand[i] = (!p.dynamic[i] && i != N - 1) ? 1 : 0;
      f.cb_forced[i] = (p.dynamic[i] || i == N - 1) ? 1 : 0;
    }
    int n_cand = 0;
    for (int i = 0; i < N; ++i) n_cand += f.cb_cand[i];
    f.cb_T = std::min(n_cand, (int)(((int64_t)pr->r_percent * n_cached + 99) / 100));  // ⌈R·N_cached/100⌉ (R11)
    if (!f.cb) {
      // check layer beyond the model: every layer recomputes all rows (≡ FR)
    } else if (pr->sel_override) {
      if (pr->n_sel_override <= 0 || pr->n_sel_override > N) {
        rollback();
        return fail(PIC_E_INVALID_ARG, "bad n_sel_override");
      }
      f.cb_override = true;
      for (int r = 0; r < pr->n_sel_override; ++r) {
        const int i = pr->sel_override[r];
        if (i < 0 || i >= N || (r && i <= pr->sel_override[r - 1])) {
          rollback();
          return fail(PIC_E_INVALID_ARG, "sel_override must be sorted distinct indices in [0,N)");
        }
        f.cb_sel2.push_back(i);
        f.cb_pos2.push_back(i);
        f.cb_slot2.push_back(slot_of(reqs[0].bt, i));
      }
      if (f.cb_sel2.back() != N - 1) {
        rollback();
        return fail(PIC_E_INVALID_ARG, "sel_override must contain the last row N-1");
      }
      f.M2 = pr->n_sel_override;
    } else {
      int n_forced = 0;
      for (int i = 0; i < N; ++i) n_forced += f.cb_forced[i];
      f.M2 = f.cb_T + n_forced;
    }
    if (f.cb) {
      add_tiles(f.tiles2, 0, 0, f.M2, qpt_of(e->cfg));
      f.head_map2.assign(f.M2, -1);
      f.head_map2[f.M2 - 1] = 0;
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool use_graph = pr->use_graph != 0;
  schedule_attention(e, f);
  pic_status s = run_forward(e, f, st, use_graph, pr->debug_hidden);
  if (s != PIC_OK) {
    rollback();
    return s;
  }
  const int V = e->cfg.vocab;
  bool want_host = false;
  for (int r = 0; r < n_req; ++r) {
    if (results[r].logits_dev) {
      cudaError_t ce = cudaMemcpyAsync(results[r].logits_dev, e->logits + (size_t)r * V, (size_t)V * 4,
                                       cudaMemcpyDeviceToDevice, st);
      if (ce != cudaSuccess) {
        rollback();
        return fail(PIC_E_CUDA, "logits copy: %s", cudaGetErrorString(ce));
      }
    }
    if (results[r].logits || !results[r].logits_dev) want_host = true;
  }
  e->d2h_last = 0;
  if (pr->debug_hidden) want_host = true;
  for (int r = 0; r < n_req; ++r) want_host |= results[r].selected != nullptr;
  std::vector<int32_t> cb_sel_host;
  if (f.cb && results[0].selected) {
    cb_sel_host.resize(f.M2);
    cudaError_t ce = cudaMemcpyAsync(cb_sel_host.data(), e->last_cb_sel2, (size_t)f.M2 * 4,
                                     cudaMemcpyDeviceToHost, st);
    if (ce != cudaSuccess) {
      rollback();
      return fail(PIC_E_CUDA, "selection copy: %s", cudaGetErrorString(ce));
    }
  }
  bool direct_logits = false;
  if (want_host) {
    bool any_logits = false;
    for (int r = 0; r < n_req; ++r) any_logits |= results[r].logits != nullptr;
    cudaError_t ce = cudaSuccess;
    // caller buffers in page-locked memory (cudaHostAlloc / cudaHostRegister): copy the logits straight into
    // them (one copy when they are rows of one array); pageable buffers go through the pinned staging area
    direct_logits = any_logits;
    for (int r = 0; r < n_req && direct_logits; ++r) {
      if (!results[r].logits) continue;
      cudaPointerAttributes at{};
      direct_logits = cudaPointerGetAttributes(&at, results[r].logits) == cudaSuccess && at.type == cudaMemoryTypeHost;
    }
    cudaGetLastError();  // (older runtimes report a pageable pointer as an error: do not leave it pending)
    if (any_logits) {
      bool rows = direct_logits;
      for (int r = 0; r < n_req && rows; ++r) rows = results[r].logits == results[0].logits + (size_t)r * V;
      if (rows) {
        ce = cudaMemcpyAsync(results[0].logits, e->logits, (size_t)n_req * V * 4, cudaMemcpyDeviceToHost, st);
      } else if (direct_logits) {
        for (int r = 0; r < n_req && ce == cudaSuccess; ++r)
          if (results[r].logits)
            ce = cudaMemcpyAsync(results[r].logits, e->logits + (size_t)r * V, (size_t)V * 4, cudaMemcpyDeviceToHost, st);
      } else {
        ce = cudaMemcpyAsync(e->host_logits, e->logits, (size_t)n_req * V * 4, cudaMemcpyDeviceToHost, st);
      }
      e->d2h_last += (int64_t)n_req * V * 4;
    }
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(e->host_amax, e->amax, (size_t)n_req * 4, cudaMemcpyDeviceToHost, st);
    e->d2h_last += (int64_t)n_req * 4;
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) {
      rollback();
      return fail(PIC_E_CUDA, "link: %s", cudaGetErrorString(ce));
    }
  }
  // every handle exists before any is handed out: a failed allocation leaves out_linked untouched
  std::vector<pic_linked*> handles;
  if (out_linked) {
    for (int r = 0; r < n_req; ++r) {
      pic_linked* h = new (std::nothrow) pic_linked();
      if (!h) {
        for (pic_linked* x : handles) delete x;
        rollback();
        return fail(PIC_E_OOM, "linked handle");
      }
      handles.push_back(h);
    }
  }
  for (int r = 0; r < n_req; ++r) {
    pic_link_result& res = results[r];
    res.n_tokens = reqs[r].p.N;
    res.n_selected_layer0 = cb ? reqs[r].p.N : (int)reqs[r].p.sel.size();
    res.n_selected = cb ? (f.cb ? f.M2 : reqs[r].p.N) : (int)reqs[r].p.sel.size();
    res.first_token = want_host ? e->host_amax[r] : -1;
    if (res.logits && !direct_logits) std::memcpy(res.logits, e->host_logits + (size_t)r * V, (size_t)V * 4);
    if (res.selected) {
      if (f.cb)
        std::copy(cb_sel_host.begin(), cb_sel_host.end(), res.selected);
      else if (cb)
        for (int i = 0; i < reqs[r].p.N; ++i) res.selected[i] = i;
      else
        std::copy(reqs[r].p.sel.begin(), reqs[r].p.sel.end(), res.selected);
    }
    if (out_linked) {
      pic_linked* h = handles[r];
      h->n_tokens = reqs[r].p.N;
      h->blocks = reqs[r].bt;
      h->bdelta = reqs[r].bdelta;
      h->n_shared = (int32_t)reqs[r].bt.size() - reqs[r].n_fresh;
      h->byref.assign(h->blocks.size(), 0);
      for (size_t b = 0; b < h->blocks.size() && b < reqs[r].shared.size(); ++b) h->byref[b] = reqs[r].shared[b] >= 0;
      h->n_vshared = 0;
      for (int32_t b : reqs[r].vshared) h->n_vshared += b >= 0;
      if (h->n_vshared) {
        h->vblocks.resize(h->blocks.size());
        for (size_t b = 0; b < h->blocks.size(); ++b)
          h->vblocks[b] = reqs[r].vshared[b] >= 0 ? reqs[r].vshared[b] : h->blocks[b];
      }
      out_linked[r] = h;
    } else {
      e->alloc.release(reqs[r].bt);  // stream-ordered reuse on the same stream
      for (int32_t b : reqs[r].vshared)
        if (b >= 0) e->alloc.release({b});
    }
  }
  return PIC_OK;
}

// ============================================================================ decode (f1)
extern "C" pic_status pic_decode(pic_engine* e, pic_linked* const* linked, const int32_t* tokens, int32_t n,
                                 int32_t use_graph, void* stream, pic_decode_result* results) {
  if (!e || !linked || !tokens || !results) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (n <= 0) return fail(PIC_E_EMPTY_INPUT, "no sequences");
  if (n > e->lim.max_requests) return fail(PIC_E_CAPACITY, "%d sequences exceed max_requests", n);
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine cannot decode");
  if (e->tp_size > 1 && !e->tp_connected) return fail(PIC_E_INVALID_ARG, "tensor-parallel engine: call pic_tp_connect first");
  int64_t need = 0;
  for (int b = 0; b < n; ++b) {
    if (!linked[b]) return fail(PIC_E_INVALID_ARG, "linked[%d] is NULL", b);
    for (int c = 0; c < b; ++c)
      if (linked[c] == linked[b]) return fail(PIC_E_INVALID_ARG, "linked[%d] repeats linked[%d]", b, c);
    if (tokens[b] < 0 || tokens[b] >= e->cfg.vocab) return fail(PIC_E_TOKEN, "token %d = %d out of range", b, tokens[b]);
    const int N = linked[b]->n_tokens;
    if (N + 1 > e->cfg.max_pos || N + 1 > e->lim.max_tokens)
      return fail(PIC_E_CAPACITY, "sequence %d: %d + 1 tokens exceed max_pos / max_tokens", b, N);
    if (N % 16 == 0) ++need;
  }
  if (!e->alloc.can(need)) return fail(PIC_E_CAPACITY, "pool has %zu free blocks, decode needs %lld",
                                       e->alloc.free_ids.size(), (long long)need);
  std::vector<int32_t> grown(n, -1);
  for (int b = 0; b < n; ++b)
    if (linked[b]->n_tokens % 16 == 0) {
      grown[b] = e->alloc.alloc(1)[0];
      linked[b]->blocks.push_back(grown[b]);
      linked[b]->bdelta.push_back(0);
      linked[b]->byref.push_back(0);
      if (!linked[b]->vblocks.empty()) linked[b]->vblocks.push_back(grown[b]);
    }
  auto rollback = [&]() {
    for (int b = 0; b < n; ++b)
      if (grown[b] >= 0) {
        linked[b]->blocks.pop_back();
        linked[b]->bdelta.pop_back();
        linked[b]->byref.pop_back();
        if (!linked[b]->vblocks.empty()) linked[b]->vblocks.pop_back();
        e->alloc.release({grown[b]});
      }
  };
  // one row per sequence: position N_b, K/V slot N_b of its own block table
  Fwd f;
  f.n_head = n;
  f.decode = true;
  const int qpt = qpt_of(e->cfg);
  for (int b = 0; b < n; ++b) {
    const pic_linked& h = *linked[b];
    f.seq_bt_off.push_back((int)f.bt.size());
    f.bt.insert(f.bt.end(), h.blocks.begin(), h.blocks.end());
    f.bdelta.insert(f.bdelta.end(), h.bdelta.begin(), h.bdelta.end());
    for (int32_t dl : h.bdelta) f.kv_rot |= dl != 0;
    const std::vector<int32_t>& vb = h.vblocks.empty() ? h.blocks : h.vblocks;
    f.vbt.insert(f.vbt.end(), vb.begin(), vb.end());
    f.has_vbt |= h.n_vshared > 0;
    add_tiles(f.tiles, b, b, 1, qpt);
    f.tok.push_back(tokens[b]);
    f.pos.push_back(h.n_tokens);
    f.slot.push_back(slot_of(h.blocks, h.n_tokens));
    f.seq.push_back(b);
    f.head_map.push_back(b);
  }
  f.M = n;
  f.debug_rows = 1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  schedule_attention(e, f);
  pic_status s = run_forward(e, f, st, use_graph != 0, nullptr);
  if (s != PIC_OK) {
    rollback();
    return s;
  }
  const int V = e->cfg.vocab;
  bool want_host = false;
  cudaError_t ce = cudaSuccess;
  for (int b = 0; b < n && ce == cudaSuccess; ++b) {
    if (results[b].logits_dev)
      ce = cudaMemcpyAsync(results[b].logits_dev, e->logits + (size_t)b * V, (size_t)V * 4, cudaMemcpyDeviceToDevice, st);
    if (results[b].logits || !results[b].logits_dev) want_host = true;
  }
  e->d2h_last = 0;
  if (ce == cudaSuccess && want_host) {
    bool any_logits = false;
    for (int b = 0; b < n; ++b) any_logits |= results[b].logits != nullptr;
    if (any_logits) {
      ce = cudaMemcpyAsync(e->host_logits, e->logits, (size_t)n * V * 4, cudaMemcpyDeviceToHost, st);
      e->d2h_last += (int64_t)n * V * 4;
    }
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(e->host_amax, e->amax, (size_t)n * 4, cudaMemcpyDeviceToHost, st);
    e->d2h_last += (int64_t)n * 4;
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  }
  if (ce != cudaSuccess) {
    rollback();
    return fail(PIC_E_CUDA, "decode: %s", cudaGetErrorString(ce));
  }
  for (int b = 0; b < n; ++b) {
    linked[b]->n_tokens += 1;
    results[b].n_tokens = linked[b]->n_tokens;
    results[b].next_token = want_host ? e->host_amax[b] : -1;
    if (results[b].logits) std::memcpy(results[b].logits, e->host_logits + (size_t)b * V, (size_t)V * 4);
  }
  return PIC_OK;
}

extern "C" pic_status pic_link(pic_engine* e, const pic_segment* segs, int32_t n_segs, const pic_link_params* params,
                               void* stream, pic_linked** out_linked, pic_link_result* result) {
  const pic_status st = link_impl(e, 1, &segs, &n_segs, params, stream, out_linked, result);
  if (st == PIC_OK && attn_trace_buffer()) {
    cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    attn_trace_print(g_attn_trace_ctas);
  }
  if (st == PIC_OK && chain_trace_buffer()) {
    cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    chain_trace_dump(e->cfg.n_layers / 2);
  }
  return st;
}

extern "C" pic_status pic_link_batch(pic_engine* e, int32_t n_req, const pic_segment* const* segs,
                                     const int32_t* n_segs, const pic_link_params* params, void* stream,
                                     pic_linked** out_linked, pic_link_result* results) {
  const pic_status st = link_impl(e, n_req, segs, n_segs, params, stream, out_linked, results);
  if (st == PIC_OK && attn_trace_buffer()) {
    cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    attn_trace_print(g_attn_trace_ctas);
  }
  return st;
}

// ============================================================================ exports / lifecycle
static pic_status export_rows(pic_engine* e, const std::vector<int32_t>& blocks, int n, int layer, void* k_host,
                              void* v_host, const std::vector<int32_t>* vblocks = nullptr) {
  if (vblocks && vblocks->empty()) vblocks = nullptr;
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine");
  if (layer < 0 || layer >= e->cfg.n_layers) return fail(PIC_E_INVALID_ARG, "layer out of range");
  const int Hkv = e->cfg.n_kv_heads, D = e->cfg.head_dim;
  const size_t es = e->f32 ? 4 : 2;
  const size_t row = (size_t)D * es;
  CK(cudaDeviceSynchronize());
  // one strided copy per (block, head) slab: pool [blk][Hkv][16][D] -> host [n][Hkv][D]
  for (int b = 0; b * 16 < n; ++b) {
    const int rows = std::min(16, n - b * 16);
    for (int g = 0; g < Hkv; ++g) {
      const size_t src = (size_t)layer * e->layer_stride + ((size_t)blocks[b] * Hkv + g) * 16 * D;
      const size_t dst = ((size_t)b * 16 * Hkv + g) * row;
      if (k_host)
        CK(cudaMemcpy2D(reinterpret_cast<char*>(k_host) + dst, Hkv * row, reinterpret_cast<char*>(e->Kpool) + src * es,
                        row, row, rows, cudaMemcpyDeviceToHost));
      if (v_host) {  // V from its own block when linked by reference (kv_share 2)
        const size_t vsrc = vblocks ? (size_t)layer * e->layer_stride + ((size_t)(*vblocks)[b] * Hkv + g) * 16 * D : src;
        CK(cudaMemcpy2D(reinterpret_cast<char*>(v_host) + dst, Hkv * row, reinterpret_cast<char*>(e->Vpool) + vsrc * es,
                        row, row, rows, cudaMemcpyDeviceToHost));
      }
    }
  }
  return PIC_OK;
}

extern "C" pic_status pic_linked_export(pic_engine* e, const pic_linked* h, int32_t layer, void* k_host, void* v_host) {
  if (!e || !h) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine");
  if (layer < 0 || layer >= e->cfg.n_layers) return fail(PIC_E_INVALID_ARG, "layer out of range");
  std::vector<int> idx;
  if (k_host)
    for (size_t b = 0; b < h->bdelta.size(); ++b)
      if (h->bdelta[b] != 0) idx.push_back((int)b);
  if (idx.empty()) return export_rows(e, h->blocks, h->n_tokens, layer, k_host, v_host, &h->vblocks);
  // Shared blocks (f3) hold keys at their compile positions.  Their re-based rows are produced on the
  // device by a2's kernel (kv_link, this layer only) into scratch pool blocks — the arithmetic the
  // attention kernels' K-tile rotation reproduces bit for bit — and exported from there.
  const size_t n = idx.size() * 16;
  if (3 * n > e->plan_cap_ints) return fail(PIC_E_CAPACITY, "export: %zu shared rows exceed the plan buffer", n);
  if (!e->alloc.can((int64_t)idx.size()))
    return fail(PIC_E_CAPACITY, "export of a shared-block link needs %zu free scratch blocks (pool has %zu)",
                idx.size(), e->alloc.free_ids.size());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> fresh = e->alloc.alloc((int64_t)idx.size());
  std::vector<int32_t> blocks = h->blocks;
  std::vector<int32_t> host(3 * n);
  for (size_t k = 0; k < idx.size(); ++k) {
    for (int j = 0; j < 16; ++j) {
      host[k * 16 + j] = h->blocks[idx[k]] * 16 + j;
      host[n + k * 16 + j] = fresh[k] * 16 + j;
      host[2 * n + k * 16 + j] = h->bdelta[idx[k]];
    }
    blocks[idx[k]] = fresh[k];
  }
  std::memcpy(e->plan_host, host.data(), host.size() * 4);
  cudaError_t ce = cudaMemcpy(e->plan_dev, e->plan_host, host.size() * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess)
    ce = launch_kv_link(e->Kpool, e->Vpool, e->plan_dev, e->plan_dev + n, e->plan_dev + 2 * n, (int)n, layer, 1,
                        e->layer_stride, e->cfg.n_kv_heads, e->cfg.head_dim, e->cos_t, e->sin_t, 1, 0, e->f32);
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    e->alloc.release(fresh);
    return fail(PIC_E_CUDA, "export re-base: %s", cudaGetErrorString(ce));
  }
  const pic_status s = export_rows(e, blocks, h->n_tokens, layer, k_host, v_host);
  e->alloc.release(fresh);
  return s;
}

extern "C" pic_status pic_linked_info(pic_engine* e, const pic_linked* h, int32_t* n_tokens, int32_t* block_table) {
  if (!e || !h) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (n_tokens) *n_tokens = h->n_tokens;
  if (block_table) std::copy(h->blocks.begin(), h->blocks.end(), block_table);
  return PIC_OK;
}

extern "C" pic_status pic_linked_sharing(pic_engine* e, const pic_linked* h, int32_t* n_shared, int32_t* block_delta) {
  if (!e || !h) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (n_shared) *n_shared = h->n_shared + h->n_vshared;  // K-and-V (kv_share 1) or V-only (kv_share 2) by reference
  if (block_delta) std::copy(h->bdelta.begin(), h->bdelta.end(), block_delta);
  return PIC_OK;
}

// Re-base the shared chunk-store blocks of a linked cache into blocks it owns (f3 -> copy layout), so
// that later decode steps read keys at their linked positions without re-rotating them every step.
// One a2 launch (all layers) over the rows of every shared block with Δ != 0; the arithmetic is a2's,
// so exports and decode outputs are unchanged bit for bit.
extern "C" pic_status pic_linked_materialize(pic_engine* e, pic_linked* h, void* stream) {
  if (!e || !h) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine");
  std::vector<int> idx;
  for (size_t b = 0; b < h->bdelta.size(); ++b)
    if (h->bdelta[b] != 0) idx.push_back((int)b);
  if (idx.empty()) return PIC_OK;
  const size_t n = idx.size() * 16;
  if (3 * n > e->plan_cap_ints) return fail(PIC_E_CAPACITY, "materialize: %zu rows exceed the plan buffer", n);
  if (!e->alloc.can((int64_t)idx.size()))
    return fail(PIC_E_CAPACITY, "pool has %zu free blocks, materialize needs %zu", e->alloc.free_ids.size(), idx.size());
  std::vector<int32_t> fresh = e->alloc.alloc((int64_t)idx.size());
  std::vector<int32_t> host(3 * n);
  for (size_t k = 0; k < idx.size(); ++k)
    for (int j = 0; j < 16; ++j) {
      host[k * 16 + j] = h->blocks[idx[k]] * 16 + j;          // src slot (chunk-store block)
      host[n + k * 16 + j] = fresh[k] * 16 + j;               // dst slot (owned block)
      host[2 * n + k * 16 + j] = h->bdelta[idx[k]];           // Δ
    }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // any failure after the allocation returns the fresh blocks (nothing observable changes on error)
  auto undo = [&](cudaError_t ce, const char* what) {
    e->alloc.release(fresh);
    return fail(PIC_E_CUDA, "materialize %s: %s", what, cudaGetErrorString(ce));
  };
  cudaError_t ce = cudaEventSynchronize(e->plan_ev);
  if (ce != cudaSuccess) return undo(ce, "plan event");
  std::memcpy(e->plan_host, host.data(), host.size() * 4);
  ce = cudaMemcpyAsync(e->plan_dev, e->plan_host, host.size() * 4, cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) return undo(ce, "plan copy");
  ce = cudaEventRecord(e->plan_ev, st);
  if (ce != cudaSuccess) return undo(ce, "plan event");
  ce = launch_kv_link(e->Kpool, e->Vpool, e->plan_dev, e->plan_dev + n, e->plan_dev + 2 * n, (int)n,
                                        0, e->cfg.n_layers, e->layer_stride, e->cfg.n_kv_heads, e->cfg.head_dim,
                                        e->cos_t, e->sin_t, 1, st, e->f32);
  if (ce != cudaSuccess) return undo(ce, "kv_link");
  // the chunk-store blocks lose this reference; later work on `stream` is ordered after the copy
  // (kv_share 3: owned chunk-frame blocks are re-based the same way and freed)
  std::vector<int32_t> old;
  for (size_t k = 0; k < idx.size(); ++k) {
    const int b = idx[k];
    old.push_back(h->blocks[b]);
    h->blocks[b] = fresh[k];
    h->bdelta[b] = 0;
    if (b < (int)h->byref.size() && h->byref[b]) {
      h->byref[b] = 0;
      --h->n_shared;
    }
  }
  e->alloc.release(old);
  return PIC_OK;
}

extern "C" pic_status pic_linked_release(pic_engine* e, pic_linked* h) {
  if (!e || !h) return fail(PIC_E_INVALID_ARG, "NULL argument");
  e->alloc.release(h->blocks);
  for (size_t b = 0; b < h->vblocks.size(); ++b)  // kv_share 2: the chunk-store blocks holding V
    if (h->vblocks[b] != h->blocks[b]) e->alloc.release({h->vblocks[b]});
  delete h;
  return PIC_OK;
}

extern "C" pic_status pic_cache_export(pic_engine* e, pic_cache_id id, int32_t layer, void* k_host, void* v_host) {
  if (!e) return fail(PIC_E_INVALID_ARG, "NULL engine");
  auto it = e->store.find(id);
  if (it == e->store.end()) return fail(PIC_E_MISSING_CACHE, "unknown cache id %llu", (unsigned long long)id);
  return export_rows(e, it->second.blocks, (int)it->second.tokens.size(), layer, k_host, v_host);
}

extern "C" pic_status pic_cache_info(pic_engine* e, pic_cache_id id, int32_t* n_tokens, int32_t* blocks) {
  if (!e) return fail(PIC_E_INVALID_ARG, "NULL engine");
  auto it = e->store.find(id);
  if (it == e->store.end()) return fail(PIC_E_MISSING_CACHE, "unknown cache id %llu", (unsigned long long)id);
  if (n_tokens) *n_tokens = (int32_t)it->second.tokens.size();
  if (blocks) std::copy(it->second.blocks.begin(), it->second.blocks.end(), blocks);
  return PIC_OK;
}

extern "C" pic_status pic_expire_cache(pic_engine* e, pic_cache_id id, int32_t* was_present) {
  if (!e) return fail(PIC_E_INVALID_ARG, "NULL engine");
  auto it = e->store.find(id);
  if (was_present) *was_present = it != e->store.end();
  if (it != e->store.end()) {
    e->alloc.release(it->second.blocks);
    e->store.erase(it);
  }
  return PIC_OK;
}

extern "C" pic_status pic_read_weights(pic_engine* e, int32_t which, int32_t layer, int64_t row0, int64_t nrows,
                                       void* host_out) {
  if (!e || !host_out) return fail(PIC_E_INVALID_ARG, "NULL argument");
  if (e->host_only) return fail(PIC_E_NO_DEVICE, "host-only engine");
  const pic_model_config& c = e->cfg;
  const int64_t d = c.d_model, D = c.head_dim, Hq = c.n_heads, Hkv = c.n_kv_heads, F = c.ffn_dim;
  if (which <= 6 && (layer < 0 || layer >= c.n_layers)) return fail(PIC_E_INVALID_ARG, "layer out of range");
  const char* base = nullptr;
  int64_t rows = 0, cols = 0;
  const LayerW* w = which <= 6 || which == 9 || which == 10 ? &e->layers[std::max(0, std::min(layer, c.n_layers - 1))]
                                                            : nullptr;
  switch (which) {
    case 0: base = (const char*)w->qkv; rows = Hq * D; cols = d; break;
    case 1: base = (const char*)w->qkv + Hq * D * d * 2; rows = Hkv * D; cols = d; break;
    case 2: base = (const char*)w->qkv + (Hq + Hkv) * D * d * 2; rows = Hkv * D; cols = d; break;
    case 3: base = (const char*)w->o; rows = d; cols = Hq * D; break;
    case 4: base = (const char*)w->gu; rows = F; cols = d; break;
    case 5: base = (const char*)w->gu + F * d * 2; rows = F; cols = d; break;
    case 6: base = (const char*)w->down; rows = d; cols = F; break;
    case 7: base = (const char*)e->E; rows = c.vocab; cols = d; break;
    case 8: base = (const char*)e->Wlm; rows = c.vocab; cols = d; break;
    case 9: CK(cudaMemcpy(host_out, w->g1, d * 4, cudaMemcpyDeviceToHost)); return PIC_OK;
    case 10: CK(cudaMemcpy(host_out, w->g2, d * 4, cudaMemcpyDeviceToHost)); return PIC_OK;
    case 11: CK(cudaMemcpy(host_out, e->gf, d * 4, cudaMemcpyDeviceToHost)); return PIC_OK;
    default: return fail(PIC_E_INVALID_ARG, "bad weight id %d", which);
  }
  if (row0 < 0 || nrows < 0 || row0 + nrows > rows) return fail(PIC_E_INVALID_ARG, "row range out of bounds");
  CK(cudaDeviceSynchronize());
  if ((which == 4 || which == 5) && e->gu_group > 0) {
    const int64_t g = e->gu_group;
    for (int64_t r = 0; r < nrows; ++r) {
      const int64_t f = row0 + r;
      const int64_t p = (f / g) * 2 * g + f % g + (which == 5 ? g : 0);
      CK(cudaMemcpy(reinterpret_cast<char*>(host_out) + r * cols * 2, (const char*)w->gu + p * cols * 2, cols * 2,
                    cudaMemcpyDeviceToHost));
    }
    return PIC_OK;
  }
  CK(cudaMemcpy(host_out, base + row0 * cols * 2, nrows * cols * 2, cudaMemcpyDeviceToHost));
  return PIC_OK;
}

static pic_status prof_push(pic_engine* e, cudaStream_t st, const char* name, double bytes, double flops,
                            bool begin) {
  cudaEvent_t ev;
  if (e->ev_pool_next < e->ev_pool.size()) {
    ev = e->ev_pool[e->ev_pool_next];
  } else {
    CK(cudaEventCreate(&ev));
    e->ev_pool.push_back(ev);
  }
  ++e->ev_pool_next;
  CK(cudaEventRecord(ev, st));
  if (begin) {
    e->prof_pending.push_back({name, ev, nullptr, bytes, flops});
  } else {
    e->prof_pending.back().end = ev;
  }
  return PIC_OK;
}

extern "C" pic_status pic_set_profiling(pic_engine* e, int32_t on) {
  if (!e) return fail(PIC_E_INVALID_ARG, "NULL engine");
  e->profiling = on != 0;
  return PIC_OK;
}

extern "C" pic_status pic_get_profile(pic_engine* e, pic_kernel_stat* out, int32_t cap, int32_t* n, int32_t reset) {
  if (!e || !n) return fail(PIC_E_INVALID_ARG, "NULL argument");
  for (auto& r : e->prof_pending) {
    if (!r.end) continue;
    CK(cudaEventSynchronize(r.end));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.begin, r.end));
    ProfAgg& a = e->prof_agg[r.name];
    a.launches += 1;
    a.ms += ms;
    a.bytes += r.bytes;
    a.flops += r.flops;
  }
  e->prof_pending.clear();
  e->ev_pool_next = 0;
  int i = 0;
  for (auto& kv : e->prof_agg) {
    if (out && i < cap) {
      std::memset(&out[i], 0, sizeof(pic_kernel_stat));
      std::snprintf(out[i].name, sizeof out[i].name, "%s", kv.first.c_str());
      out[i].launches = kv.second.launches;
      out[i].ms = kv.second.ms;
      out[i].bytes = kv.second.bytes;
      out[i].flops = kv.second.flops;
    }
    ++i;
  }
  *n = i;
  if (reset) e->prof_agg.clear();
  return PIC_OK;
}

extern "C" pic_status pic_get_stats(pic_engine* e, pic_stats* out) {
  if (!e || !out) return fail(PIC_E_INVALID_ARG, "NULL argument");
  out->free_blocks = (int64_t)e->alloc.free_ids.size();
  out->total_blocks = e->lim.num_blocks;
  out->n_cached_chunks = (int64_t)e->store.size();
  out->kernels_last_call = e->kernels_last;
  out->graphs_cached = (int64_t)e->graphs.size();
  out->h2d_bytes_last_call = e->h2d_last;
  out->d2h_bytes_last_call = e->d2h_last;
  return PIC_OK;
}
