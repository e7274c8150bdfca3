// runtime.cu — the C ABI (include/dhen.h) and the DHEN layer-stack runtime:
// config validation, canonical parameter layout, carving of caller-provided
// memory, per-layer forward/backward as sequences of our kernels, head + loss,
// SGD, and FSDP parameter all-gather / gradient reduce-scatter over NCCL.
//
// Forward of layer n (Eq.(1)(2)): each module
// writes its l_i output tokens into an fp32 concat buffer Ucat at token offset
// sum_{j<i} l_j; the shortcut (W_n^T X when the token counts differ) is
// accumulated into Ucat; the LN kernel adds the identity shortcut, normalises
// and writes Y.  Backward mirrors it (B1-B12).  bf16 storage points are listed
// in DESIGN.md §4 and mirrored by the oracle's Precision.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dhen.h"
#include "../../include/dhen_debug.h"
#include "gemm.h"
#include "kernels.h"
#include "attn.h"
#include "dot_bwd.h"
#include "dcn_bwd.h"
#include "comm.h"
#include "tuning.h"

using namespace dhen;

// ------------------------------------------------------------------ errors
static thread_local std::string t_err;
static dhen_status fail(dhen_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return s;
}
namespace dhen {
dhen_status fail_msg(dhen_status s, const char* msg) {   // the error of a call outside this file (fp.cu)
  t_err = msg;
  return s;
}
}  // namespace dhen
#define CK(call)                                                                               \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return fail(DHEN_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define NK(call)                                                                               \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess) return fail(DHEN_E_NCCL, "%s: %s", #call, ncclGetErrorString(r_));  \
  } while (0)
#define RET(call)                         \
  do {                                    \
    dhen_status s_ = (call);              \
    if (s_ != DHEN_OK) return s_;         \
  } while (0)

// ------------------------------------------------------------------ plan structures
namespace {

struct Mod {
  dhen_module s;
  int off_tok = 0;   // token offset of this module's outputs in the concat
  // parameter offsets inside the layer group (canonical order)
  int64_t W = -1, b = -1, Wu = -1, Wm = -1, K = -1;
  int64_t Wq = -1, Wo = -1, bq = -1, bv = -1, bo = -1, g1 = -1, be1 = -1, g2 = -1, be2 = -1, W1 = -1, b1 = -1, W2 = -1, b2 = -1;
  // saved activations (work)
  void *Z = nullptr, *A = nullptr, *T = nullptr, *QKV = nullptr, *P = nullptr, *O = nullptr, *R1 = nullptr,
       *Z1 = nullptr, *F = nullptr, *R2 = nullptr, *h1 = nullptr, *h2 = nullptr;
  float *mu1 = nullptr, *rs1 = nullptr, *mu2 = nullptr, *rs2 = nullptr;
  void* bdT = nullptr;   // bf16 [128][spt m]: blockdiag(W_u^T, ..) for the packed token projection (layer LN fused)
  void* bdg = nullptr;   // bf16 [128][128]: blockdiag(W_u, ..) for the packed DCN backward dT
  // backward scratch of its own (not the shared tA / tC), so the module's data gradients never wait for an
  // earlier module's side-stream weight gradients: MLP dh2 / dh1, Conv dT
  void *dh2 = nullptr, *dh1 = nullptr, *dT = nullptr;
  void *G = nullptr, *S = nullptr;   // paper-literal DCN: saved d x d Gram per sample (dt), symmetrised dG (dt)
  float* dGf = nullptr;              //                    dG (fp32 scratch)
  float* Uo = nullptr;   // sum / weighted-sum ensembles: this module's output U_i (fp32 [B][m_out][d], saved)
  void* dUs = nullptr;   // weighted sum: this module's dU_i = bf16(w_i dR)
  bool bdT_pre = false, bdg_pre = false;   // built for this step by prebuild_bd (train_step, one launch)
  uint32_t* Fbits = nullptr;   // attention FFN ReLU bitmask [f / 32][B m] (FFN2 data gradient reads it, not F)
};

struct Group {
  int64_t n = 0, npad = 0, shard = 0;   // numel, padded numel, per-rank shard
  float* master = nullptr;              // fp32 [shard] (the full vector when world == 1 / DP)
  void* comp = nullptr;                 // dtype copy [shard] (full when world == 1 / DP)
  float* grad = nullptr;                // fp32 [npad] full gradient (accumulated in bwd)
  float* gshard = nullptr;              // fp32 [shard] reduced gradient shard (world > 1)
  float *adam_m = nullptr, *adam_v = nullptr;   // Adam moments [shard] (cfg.optimizer 1: fp32; 2: bf16 storage)
  std::vector<int64_t> toff, tn;        // tensors: internal offset (64-element aligned), numel
  std::vector<int64_t> tcanon;          // tensors: offset in the dense canonical order (params_io)
  int64_t ncanon = 0;                   // canonical (dense) numel
  std::vector<int> tinit;               // 0 uniform, 1 ones, 2 zeros
  std::vector<float> tbound;
};

struct Layer {
  int m_in = 0, m_out = 0;
  int m_mod = 0;             // tokens the modules read: m_in, + dense_tokens with dense injection (R38)
  bool inj = false;          // dense_in: modules read [X_n ; D]
  void* Xin = nullptr;       // inj: the widened module input [B][m_mod][d] (work)
  const void* Xs = nullptr;  // forward input X_n (the shortcut's; Xs == X without injection)
  int ens = 0;               // dhen_ensemble
  std::vector<Mod> mods;
  int64_t Wn = -1, gamma = -1, beta = -1, ensw = -1;
  void* Y = nullptr;
  void* R = nullptr;
  float *mu = nullptr, *rstd = nullptr;
  const void* X = nullptr;   // forward input (referenced)
  int B = -1;                // batch of the saved forward, -1 = none
};

struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base((char*)b) {}
  void* take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    void* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  }
};

}  // namespace

struct dhen_ctx {
  dhen_config cfg;
  std::vector<dhen_layer> layers_cfg;
  std::vector<std::vector<dhen_module>> mods_cfg;
  dhen_dist dist;
  int dt, es;            // storage dtype, element size
  int d, Bmax;
  std::vector<Layer> L;
  std::vector<Group> G;  // n_layers + 1 (head)
  // gathered compute copies (world > 1, FSDP): 2 ping-pong buffers of max npad
  void* gathered[2] = {nullptr, nullptr};
  int gathered_owner[2] = {-1, -1};
  int64_t max_npad = 0;
  // scratch
  float* Ucat = nullptr;
  float* dXacc = nullptr;
  float* dXacc2 = nullptr;        // R38: the modules' dX accumulator of injected layers [B][m_mod][d] (fp32)
  float* dD = nullptr;            // R38: the injected dense tokens' gradient, summed over layers [B][nD][d]
  bool dense_active = false;      // some layer injects dense tokens
  const void* x0_cur = nullptr;   // X0 of the current step (layer 0's forward input): the injected tokens' source
  void* dR = nullptr;
  void* dY[2] = {nullptr, nullptr};
  dhen_tuning tune = tuning_default();   // schedule / fusion switches of this context (dhen_debug.h)
  float* big = nullptr;     // fp32 scratch [B*H*m*m] / [B*m*m] (Gram, attention S / dP)
  void* tA = nullptr;       // dtype scratch [B * m * d * 3] (dT, dQKV, ...)
  void* tB = nullptr;       // dtype scratch [B * m * d]
  void* tC = nullptr;       // dtype scratch [B * m * max(f, d)] (dF, dh*)
  void* tE = nullptr;       // dtype scratch [B * m * d]: attention dO (its own buffer: side-stream readers of dR2)
  void* tF = nullptr;       // dtype scratch [B * m * 3d]: attention dQKV (its own buffer: side-stream readers of dF)
  void* tD = nullptr;       // dtype scratch [B * H * m * m] (dS, S of Dot bwd)
  void* bdiag = nullptr;    // bf16 [128][128]: blockdiag(W_u, ..) for several samples per 128-row tile
  float* rtmp = nullptr;    // fp32 [B * m * d]
  float* red = nullptr;     // reduction partials
  size_t red_bytes = 0;
  Workspace ws;
  // weight-gradient side stream (B4/B5/B7/B8/B9 wgrads overlap the same module's dgrads; joined per module)
  cudaStream_t side_st = nullptr;
  cudaEvent_t ev_sf = nullptr, ev_sx = nullptr, ev_sj = nullptr, ev_red = nullptr;
  Workspace ws2;                      // split-K scratch of the side stream
  float* red2 = nullptr;              // reduction scratch of the side stream
  float* red3 = nullptr;              // layer-LN parameter partials (their final sum trails on the side stream)
  float* bsum = nullptr;              // DCN backward: per-CTA column sums of dA from the dT GEMM epilogue
  float* csum = nullptr;              // attention FFN: 32-row column sums of dF from the FFN2 dgrad epilogue
  bool vdy_now = false;               // set by train_step for the last layer's backward
  float *pooled = nullptr, *z = nullptr, *lossb = nullptr, *dz = nullptr;
  void* headw = nullptr;    // FSDP: the gathered head weight w_h, kept for the last layer's in-LN dY (vdy)
  int* adam_t = nullptr;    // Adam: completed optimizer steps (device; the next update is step *adam_t + 1)
  float* gtmp = nullptr;    // fp32 [max_npad]: all-gather target of params_io / grads_get (world > 1)
  void* gbf[2] = {nullptr, nullptr};   // bf16 reduce-scatter: [max_npad] bf16 gradient send buffers (ping-pong)
  void* gbf_shard = nullptr;           //                      [max shard] bf16 receive buffer
  cudaEvent_t ev_rs[2] = {nullptr, nullptr};   // the reduce-scatter that read gbf[k] has finished
  Comm* comm = nullptr;                // collectives (world > 1): NCCL or the in-process loopback (comm.h)
  // CUDA graph of dhen_train_step (dhen_train_step_graphed), keyed by its arguments
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_st = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  const void* gkey[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  int gkey_B = 0, gkey_Bg = 0;
  float gkey_lr = 0.f;
  unsigned long long graph_launches = 0;   // kernels inside the captured step
  // dhen_train_step_host: two host->device staging slots (copy stream), the step's input buffers, the loss
  void* hx[2] = {nullptr, nullptr};
  float* hy[2] = {nullptr, nullptr};
  void* hxin = nullptr;
  float* hyin = nullptr;
  float* hloss = nullptr;
  cudaStream_t hcp = nullptr;
  cudaEvent_t hev_up[2] = {nullptr, nullptr}, hev_free[2] = {nullptr, nullptr};
  unsigned long long hcalls = 0;
  cudaStream_t comm_st = nullptr;     // collectives (world > 1)
  cudaEvent_t ev_ag[2] = {nullptr, nullptr}, ev_use[2] = {nullptr, nullptr}, ev_grad = nullptr, ev_comm = nullptr;
  cudaEvent_t ev_grad2 = nullptr, ev_cfork = nullptr;
  bool graph_off = false;             // world > 1: capturing the step failed once -> eager steps from then on
  unsigned long long launches0 = 0;
  // per-op device timing (dhen_profile): event pairs on the launch stream
  struct Rec { const char* tag; int e0, e1; double flops, bytes; int tc; cudaStream_t st; };
  bool prof = false;
  int prof_mode = 1;   // dhen_profile: 1 serialised side stream, 2 concurrency kept
  std::vector<cudaEvent_t> events;
  int next_event = 0;
  std::vector<Rec> recs;
};

// The profiled pass runs serialised (every op's event-timed duration is its own) unless dhen_profile(ctx, 2)
// keeps the side stream (the dhen_debug_profile_trace timeline then shows the real concurrency).
static bool serial_prof(const dhen_ctx* c) { return c->prof && c->prof_mode != 2; }
// RAII scope recording a CUDA event pair around one op when profiling is on.
// Per-op scope: an NVTX range named after the op (so `ncu --nvtx --nvtx-include "<op>/"` captures exactly that
// op's kernels; a no-op without an attached tool) and, in profiling mode, CUDA events around the op.
struct ProfScope {
  dhen_ctx* c;
  cudaStream_t st;
  int rec = -1;
  ProfScope(dhen_ctx* c_, const char* tag, double flops, double bytes, cudaStream_t st_) : c(c_), st(st_) {
    nvtxRangePushA(tag);
    if (!c->prof) return;
    if (c->next_event + 2 > (int)c->events.size()) {
      if (c->events.size() >= (1u << 16)) return;   // pool exhausted: stop recording
      size_t n0 = c->events.size();
      c->events.resize(n0 + 1024);
      for (size_t i = n0; i < c->events.size(); ++i) cudaEventCreate(&c->events[i]);
    }
    int e0 = c->next_event++, e1 = c->next_event++;
    cudaEventRecord(c->events[e0], st);
    c->recs.push_back({tag, e0, e1, flops, bytes, 0, st});
    rec = (int)c->recs.size() - 1;
  }
  ~ProfScope() {
    if (rec >= 0) cudaEventRecord(c->events[c->recs[rec].e1], st);
    nvtxRangePop();
  }
};
#define KT(tag, flops, bytes, call)                          \
  do {                                                       \
    ProfScope ps_(c, tag, (double)(flops), (double)(bytes), st); \
    CK(call);                                                \
  } while (0)
// the same on an explicit stream (the weight-gradient side stream)
#define KTS(strm, tag, flops, bytes, call)                   \
  do {                                                       \
    ProfScope ps_(c, tag, (double)(flops), (double)(bytes), strm); \
    CK(call);                                                \
  } while (0)

// ------------------------------------------------------------------ validation / planning
static int mdef(int v, int d) { return v > 0 ? v : d; }

static dhen_status validate(const dhen_config* c) {
  if (!c) return fail(DHEN_E_CONFIG, "dhen_validate: cfg is NULL");
  if (c->m0 < 1 || c->d < 1 || c->n_layers < 1 || !c->layers)
    return fail(DHEN_E_CONFIG, "dhen_validate: m0=%d d=%d n_layers=%d layers=%p", c->m0, c->d, c->n_layers, (void*)c->layers);
  if (c->d % 8 != 0) return fail(DHEN_E_CONFIG, "dhen_validate: d=%d not a multiple of 8 (16-byte rows)", c->d);
  if (c->d > 1024) return fail(DHEN_E_CONFIG, "dhen_validate: d=%d > 1024", c->d);
  if (c->dtype != DHEN_FP32 && c->dtype != DHEN_BF16) return fail(DHEN_E_CONFIG, "dhen_validate: dtype=%d", c->dtype);
  if (c->batch_max_local < 1) return fail(DHEN_E_CONFIG, "dhen_validate: batch_max_local=%d", c->batch_max_local);
  if (c->optimizer < 0 || c->optimizer > 2)
    return fail(DHEN_E_CONFIG, "dhen_validate: optimizer=%d (0 SGD, 1 Adam, 2 Adam with bf16 moments)", c->optimizer);
  int m = c->m0;
  if (c->dense_tokens < 0 || c->dense_tokens > c->m0)
    return fail(DHEN_E_CONFIG, "dhen_validate: dense_tokens=%d (0 .. m0=%d)", c->dense_tokens, c->m0);
  for (int n = 0; n < c->n_layers; ++n) {
    const dhen_layer& L = c->layers[n];
    if (L.n_modules < 1 || !L.modules) return fail(DHEN_E_CONFIG, "dhen_validate: layer %d has no modules", n);
    if (L.dense_in && c->dense_tokens < 1)
      return fail(DHEN_E_CONFIG, "dhen_validate: layer %d injects dense tokens but dense_tokens=0 (R38)", n);
    const int m_layer = m;
    if (L.dense_in) m += c->dense_tokens;   // the modules read m_in + dense_tokens tokens
    int mo = 0;
    if (L.ensemble < DHEN_CONCAT || L.ensemble > DHEN_WSUM)
      return fail(DHEN_E_CONFIG, "dhen_validate: layer %d ensemble=%d (0 concat, 1 sum, 2 weighted sum)", n, L.ensemble);
    for (int i = 0; i < L.n_modules; ++i) {
      const dhen_module& s = L.modules[i];
      if (L.ensemble != DHEN_CONCAT && s.l != L.modules[0].l)
        return fail(DHEN_E_CONFIG, "dhen_validate: layer %d sum ensemble with l=%d and l=%d (P:91 needs equal l_i)", n,
                    L.modules[0].l, s.l);
      if (s.kind < DHEN_DOT || s.kind > DHEN_DCN_FULL) return fail(DHEN_E_CONFIG, "dhen_validate: layer %d module %d kind=%d", n, i, s.kind);
      if (s.l < 1) return fail(DHEN_E_CONFIG, "dhen_validate: layer %d module %d l=%d < 1", n, i, s.l);
      if (s.kind == DHEN_DOT && m < 2) return fail(DHEN_E_CONFIG, "dhen_validate: layer %d Dot needs m >= 2, m=%d (S:186)", n, m);
      if (s.kind == DHEN_ATTN && c->d % mdef(s.heads, 2) != 0)
        return fail(DHEN_E_CONFIG, "dhen_validate: layer %d attention d=%d %% heads=%d != 0 (S:195)", n, c->d, mdef(s.heads, 2));
      if (s.kind == DHEN_CONV && (mdef(s.conv_k, 3) % 2 == 0 || mdef(s.conv_k, 3) > 7))
        return fail(DHEN_E_CONFIG, "dhen_validate: layer %d conv_k=%d must be odd and <= 7 (S:204)", n, mdef(s.conv_k, 3));
      mo += s.l;
    }
    if (L.ensemble != DHEN_CONCAT) mo = L.modules[0].l;
    (void)m_layer;
    m = mo;
  }
  return DHEN_OK;
}

// Builds layer/group structure; carves state/work when the carvers have bases.
static void plan(dhen_ctx* c, Carver& state, Carver& work) {
  const int d = c->d, B = c->Bmax, es = c->es;
  const int world = c->dist.world;
  const bool shard = world > 1 && c->dist.fsdp;
  int m = c->cfg.m0, m_max = m, H_mm_max = 0, f_max = d, m_out_max = 0;
  int64_t tC_elems = 0, tA_elems = 0, csum_elems = 0, fsh_elems = 0, fbsh_words = 0;
  bool has_attn_any = false;
  for (int n = 0; n < c->cfg.n_layers; ++n)
    for (int i = 0; i < c->cfg.layers[n].n_modules; ++i) has_attn_any |= c->cfg.layers[n].modules[i].kind == DHEN_ATTN;
  c->L.assign(c->cfg.n_layers, Layer());
  c->G.assign(c->cfg.n_layers + 1, Group());
  for (int n = 0; n < c->cfg.n_layers; ++n) {
    Layer& Lr = c->L[n];
    Group& g = c->G[n];
    const dhen_layer& lc = c->cfg.layers[n];
    Lr.m_in = m;
    Lr.inj = lc.dense_in != 0;
    Lr.m_mod = m + (Lr.inj ? c->cfg.dense_tokens : 0);
    int mo = 0;
    for (int i = 0; i < lc.n_modules; ++i) mo += lc.modules[i].l;
    Lr.ens = lc.ensemble;
    if (Lr.ens != DHEN_CONCAT) mo = lc.modules[0].l;
    Lr.m_out = mo;
    int64_t off = 0;
    int64_t coff = 0;
    auto tensor = [&](int64_t numel, int init, int fan) {
      off = (off + 63) / 64 * 64;   // every tensor starts 128-B aligned (TMA / vector access)
      int64_t o = off;
      g.toff.push_back(off);
      g.tcanon.push_back(coff);
      coff += numel;
      g.tn.push_back(numel);
      g.tinit.push_back(init);
      g.tbound.push_back(fan > 0 ? 1.f / sqrtf((float)fan) : 0.f);
      off += numel;
      return o;
    };
    Lr.mods.clear();
    int tok = 0;
    const int m_layer = m;
    m = Lr.m_mod;   // module parameters are shaped by the tokens the modules read (R38)
    for (int i = 0; i < lc.n_modules; ++i) {
      Mod md;
      md.s = lc.modules[i];
      md.s.heads = mdef(md.s.heads, 2);
      md.s.ffn_mult = mdef(md.s.ffn_mult, 4);
      md.s.conv_channels = mdef(md.s.conv_channels, 4);
      md.s.conv_k = mdef(md.s.conv_k, 3);
      md.s.mlp_hidden[0] = mdef(md.s.mlp_hidden[0], 1024);
      md.s.mlp_hidden[1] = mdef(md.s.mlp_hidden[1], 1024);
      md.off_tok = Lr.ens == DHEN_CONCAT ? tok : 0;   // sum ensembles: every module covers all m_out tokens
      tok += md.s.l;
      const int l = md.s.l;
      switch (md.s.kind) {
        case DHEN_DOT: { int h = m * (m - 1) / 2; md.Wm = tensor((int64_t)l * d * h, 0, h); break; }
        case DHEN_LINEAR: md.W = tensor((int64_t)m * l, 0, m); break;
        case DHEN_DCN: md.W = tensor((int64_t)d * d, 0, d); md.b = tensor(d, 0, d); md.Wu = tensor((int64_t)m * l, 0, m); break;
        case DHEN_DCN_FULL: {   // R37: the cross over the flattened sample, W [m d][m d]
          const int64_t f = (int64_t)m * d;
          md.W = tensor(f * f, 0, (int)f); md.b = tensor(f, 0, (int)f); md.Wu = tensor((int64_t)m * l, 0, m);
          break;
        }
        case DHEN_CONV: { int k = md.s.conv_k; md.K = tensor((int64_t)md.s.conv_channels * k * k, 0, k * k); md.Wu = tensor((int64_t)m * l, 0, m); break; }
        case DHEN_ATTN: {
          int f = md.s.ffn_mult * d;
          md.Wq = tensor((int64_t)d * d, 0, d); tensor((int64_t)d * d, 0, d); tensor((int64_t)d * d, 0, d);
          md.Wo = tensor((int64_t)d * d, 0, d);
          md.bq = tensor(d, 0, d); md.bv = tensor(d, 0, d); md.bo = tensor(d, 0, d);
          md.g1 = tensor(d, 1, 0); md.be1 = tensor(d, 2, 0); md.g2 = tensor(d, 1, 0); md.be2 = tensor(d, 2, 0);
          md.W1 = tensor((int64_t)f * d, 0, d); md.b1 = tensor(f, 0, d); md.W2 = tensor((int64_t)d * f, 0, f); md.b2 = tensor(d, 0, f);
          md.Wu = tensor((int64_t)m * l, 0, m);
          break;
        }
        case DHEN_DCN_LIT: md.W = tensor((int64_t)d * l, 0, d); md.b = tensor((int64_t)l * d, 0, d); break;
        case DHEN_MLP: {
          int h1 = md.s.mlp_hidden[0], h2 = md.s.mlp_hidden[1];
          md.W1 = tensor((int64_t)h1 * m * d, 0, m * d); md.b1 = tensor(h1, 0, m * d);
          md.W2 = tensor((int64_t)h2 * h1, 0, h1); md.b2 = tensor(h2, 0, h1);
          md.Wm = tensor((int64_t)l * d * h2, 0, h2);
          break;
        }
      }
      Lr.mods.push_back(md);
    }
    m = m_layer;
    m_max = std::max(m_max, Lr.m_mod);
    if (Lr.ens == DHEN_WSUM) Lr.ensw = tensor(lc.n_modules, 1, 0);   // R27: initialised to 1
    if (m != mo) Lr.Wn = tensor((int64_t)m * mo, 0, m);
    Lr.gamma = tensor(d, 1, 0);
    Lr.beta = tensor(d, 2, 0);
    g.n = off;
    g.ncanon = coff;
    m = mo;
    m_max = std::max(m_max, mo);
    m_out_max = std::max(m_out_max, mo);
  }
  {  // head group (R17)
    Group& g = c->G[c->cfg.n_layers];
    const int64_t bo = (d + 63) / 64 * 64;
    g.toff = {0, bo}; g.tn = {d, 1}; g.tinit = {0, 0}; g.tcanon = {0, d};
    g.tbound = {1.f / sqrtf((float)d), 1.f / sqrtf((float)d)};
    g.n = bo + 1;
    g.ncanon = d + 1;
  }
  // sizes of every group, then state memory
  c->max_npad = 0;
  for (auto& g : c->G) {
    int64_t q = (int64_t)64 * (shard ? world : 1);
    g.npad = (g.n + q - 1) / q * q;
    g.shard = shard ? g.npad / world : g.npad;
    c->max_npad = std::max(c->max_npad, g.npad);
    g.master = (float*)state.take(g.shard * 4);
    g.comp = state.take(g.shard * es);
    g.grad = (float*)state.take(g.npad * 4);
    g.gshard = world > 1 ? (float*)state.take(g.shard * 4) : nullptr;
    if (c->cfg.optimizer >= 1) {   // Adam moments: fp32 (1) or bf16 (2, the BF16 optimizer of R35)
      g.adam_m = (float*)state.take(g.shard * (c->cfg.optimizer == 2 ? 2 : 4));
      g.adam_v = (float*)state.take(g.shard * (c->cfg.optimizer == 2 ? 2 : 4));
    }
  }
  if (c->cfg.optimizer >= 1) c->adam_t = (int*)state.take(256);
  if (shard) { c->gathered[0] = state.take(c->max_npad * es); c->gathered[1] = state.take(c->max_npad * es); }
  if (world > 1) c->gtmp = (float*)state.take(c->max_npad * 4);
  if (world > 1 && c->dist.grad_bf16) {
    c->gbf[0] = state.take(c->max_npad * 2);
    c->gbf[1] = state.take(c->max_npad * 2);
    c->gbf_shard = state.take(c->max_npad * 2);
  }
  // saved activations (work)
  m = c->cfg.m0;
  for (int n = 0; n < c->cfg.n_layers; ++n) {
    Layer& Lr = c->L[n];
    const int mi = Lr.m_mod, mo = Lr.m_out;   // (module buffers: the tokens the modules read)
    if (Lr.inj) Lr.Xin = work.take((size_t)B * mi * d * es);
    Lr.Y = work.take((size_t)B * mo * d * es);
    Lr.R = work.take((size_t)B * mo * d * es);
    Lr.mu = (float*)work.take((size_t)B * mo * 4);
    Lr.rstd = (float*)work.take((size_t)B * mo * 4);
    for (Mod& md : Lr.mods) {
      size_t tok = (size_t)B * mi * d;
      switch (md.s.kind) {
        case DHEN_DOT:
          md.Z = work.take((size_t)B * (mi * (mi - 1) / 2) * es);
          H_mm_max = std::max(H_mm_max, mi * mi);
          tA_elems = std::max<int64_t>(tA_elems, (int64_t)B * (mi * (mi - 1) / 2));
          break;
        case DHEN_DCN: case DHEN_DCN_FULL: md.A = work.take(tok * es); md.T = work.take(tok * es); break;
        case DHEN_DCN_LIT:
          md.G = work.take((size_t)B * d * d * es);
          md.S = work.take((size_t)B * d * d * es);
          md.dGf = (float*)work.take((size_t)B * d * d * 4);
          break;
        case DHEN_CONV: md.T = work.take(tok * es); md.dT = work.take(tok * es); break;
        case DHEN_ATTN: {
          int H = md.s.heads, f = md.s.ffn_mult * d;
          md.QKV = work.take(tok * 3 * es);
          const int mp = (mi + 7) / 8 * 8;   // score rows padded to 16 B (TMA pitch)
          md.P = work.take((size_t)B * H * mi * mp * es);
          md.O = work.take(tok * es);
          md.R1 = work.take(tok * es);
          md.Z1 = work.take(tok * es);
          if (c->cfg.recompute & 1) {   // shared across layers (assigned below); recomputed by the backward
            fsh_elems = std::max<int64_t>(fsh_elems, (int64_t)B * mi * f);
            fbsh_words = std::max<int64_t>(fbsh_words, (int64_t)B * mi * ((f + 31) / 32));
          } else {
            md.F = work.take((size_t)B * mi * f * es);
            md.Fbits = (uint32_t*)work.take((size_t)B * mi * ((f + 31) / 32) * 4);
          }
          md.R2 = work.take(tok * es);
          md.T = work.take(tok * es);
          md.mu1 = (float*)work.take((size_t)B * mi * 4); md.rs1 = (float*)work.take((size_t)B * mi * 4);
          md.mu2 = (float*)work.take((size_t)B * mi * 4); md.rs2 = (float*)work.take((size_t)B * mi * 4);
          H_mm_max = std::max(H_mm_max, H * mi * mp);
          f_max = std::max(f_max, f);
          tC_elems = std::max<int64_t>(tC_elems, (int64_t)B * mi * std::max(f, 3 * d));
          csum_elems = std::max<int64_t>(csum_elems, ((int64_t)B * mi + 31) / 32 * f);
          break;
        }
        case DHEN_MLP: {
          md.h1 = work.take((size_t)B * md.s.mlp_hidden[0] * es);
          md.h2 = work.take((size_t)B * md.s.mlp_hidden[1] * es);
          md.dh2 = work.take((size_t)B * md.s.mlp_hidden[1] * es);
          md.dh1 = work.take((size_t)B * md.s.mlp_hidden[0] * es);
          tC_elems = std::max<int64_t>(tC_elems, (int64_t)B * std::max(md.s.mlp_hidden[0], md.s.mlp_hidden[1]));
          tA_elems = std::max<int64_t>(tA_elems, (int64_t)B * md.s.mlp_hidden[1]);
          break;
        }
        default: break;
      }
      md.bdT = work.take((size_t)128 * 128 * 8 * 2);   // spt m <= 1024 columns
      if (Lr.ens != DHEN_CONCAT) md.Uo = (float*)work.take((size_t)B * mo * d * 4);
      if (Lr.ens == DHEN_WSUM) md.dUs = work.take((size_t)B * mo * d * es);
      if (md.s.kind == DHEN_DCN || md.s.kind == DHEN_DCN_FULL) md.bdg = work.take((size_t)128 * 128 * 2);
    }
  }
  if (fsh_elems) {   // recompute: one F / bitmask buffer for every attention module
    void* F = work.take((size_t)fsh_elems * es);
    uint32_t* Fb = (uint32_t*)work.take((size_t)fbsh_words * 4);
    for (Layer& Lr : c->L)
      for (Mod& md : Lr.mods)
        if (md.s.kind == DHEN_ATTN) { md.F = F; md.Fbits = Fb; }
  }
  // scratch
  const size_t rows_d = (size_t)B * m_max * d;
  c->Ucat = (float*)work.take((size_t)B * m_out_max * d * 4);
  c->dXacc = (float*)work.take(rows_d * 4);
  c->dense_active = false;
  for (const Layer& Lr : c->L) c->dense_active = c->dense_active || Lr.inj;
  if (c->dense_active) {
    c->dXacc2 = (float*)work.take(rows_d * 4);
    c->dD = (float*)work.take((size_t)B * c->cfg.dense_tokens * d * 4);
  }
  c->dR = work.take(rows_d * es);
  c->dY[0] = work.take(rows_d * es);
  c->dY[1] = work.take(rows_d * es);
  c->big = (float*)work.take((size_t)B * std::max(H_mm_max, 1) * 4);
  c->tA = work.take((size_t)std::max<int64_t>(tA_elems, (int64_t)rows_d * 3) * es);
  c->tB = work.take(rows_d * es);
  c->tC = work.take((size_t)std::max<int64_t>(tC_elems, 1) * es);
  if (has_attn_any) {
    c->tE = work.take(rows_d * es);
    c->tF = work.take(rows_d * 3 * es);
  }
  c->tD = work.take((size_t)B * std::max(H_mm_max, 1) * es);
  c->rtmp = (float*)work.take(rows_d * 4);
  c->bdiag = work.take((size_t)128 * 128 * 2);   // block-diagonal token map (DCN backward, m <= 64)
  c->red_bytes = (size_t)16 << 20;
  c->red = (float*)work.take(c->red_bytes);
  c->ws.bytes = (size_t)256 << 20;
  c->ws.ptr = (float*)work.take(c->ws.bytes);
  c->ws2.bytes = (size_t)256 << 20;
  c->ws2.ptr = (float*)work.take(c->ws2.bytes);
  c->red2 = (float*)work.take(c->red_bytes);
  c->red3 = (float*)work.take(c->red_bytes);
  c->bsum = (float*)work.take((size_t)4 * 148 * 256 * 4);   // DCN bias partial rows [<= 592][d <= 256]
  if (csum_elems) c->csum = (float*)work.take((size_t)csum_elems * 4);   // attention db_1 partial rows
  c->pooled = (float*)work.take(((size_t)B * d + (size_t)B * (d + 2)) * 4);   // + head partials [B][d + 2]
  c->z = (float*)work.take((size_t)B * 4);
  c->lossb = (float*)work.take((size_t)B * 4);
  c->dz = (float*)work.take((size_t)B * 4);
  c->headw = work.take((size_t)d * es);
  (void)f_max;
}

// ------------------------------------------------------------------ GEMM helpers
static double vbytes(const View& v, double n) { return v.ptr ? n * (v.dt == F32 ? 4 : 2) : 0; }
// Algorithmic traffic of a GEMM: each operand read once (shared operands once), C written, and C read only
// when it is really read: `+=` (accumulate), or the DCN backward's red.global.add into the fp32 dX accumulator
// (dcn_bwd without a residual; with one, the epilogue is dX's first writer and only stores C).
static double gemm_bytes(const Gemm& g) {
  const double es = g.a.dt == F32 ? 4 : 2;
  const double mn = (double)g.M * g.N * g.batch;
  const bool c_read = g.e.accumulate || (g.e.dcn_bwd && !g.e.resid.ptr);
  return (double)g.M * g.K * es * (g.a.bs0 || g.a.bs1 ? g.batch : 1) +
         (double)g.N * g.K * es * (g.b.bs0 || g.b.bs1 ? g.batch : 1) +
         vbytes(g.c, mn) * (c_read ? 2 : 1) + vbytes(g.e.resid, mn) + vbytes(g.e.mask, mn) +
         (g.e.cross.ptr == g.a.ptr ? 0.0 : vbytes(g.e.cross, mn)) + vbytes(g.e.aux, mn);   // (the DCN cross reads X
                                                                                              //  as A and as cross: once)
}
static inline dhen_status G_(const Gemm& g, dhen_ctx* c, cudaStream_t st, const char* tag, const Workspace* ws = nullptr) {
  const double bytes = gemm_bytes(g);
  ProfScope ps(c, tag, 2.0 * (double)g.M * g.N * g.K * g.batch, bytes, st);
  CK(gemm_run(g, ws ? *ws : (st == c->side_st ? c->ws2 : c->ws), st));   // each stream its own split-K scratch
  if (ps.rec >= 0) c->recs[ps.rec].tc = g_last_gemm_tc;
  return DHEN_OK;
}
// The DCN backward dT GEMM with the fused dA column sums (Epilogue::bsum) when its tcgen05 pass can take
// them; otherwise the same GEMM without (and *rows = 0: the caller sums dA with colsum_add instead).
// `overlap` = bytes of an operand that lie inside another counted view (the dU slice of the dR residual:
// read once), subtracted from the algorithmic bytes.
static dhen_status G_dT(Gemm& g, dhen_ctx* c, cudaStream_t st, int* rows, double overlap) {
  *rows = 0;
  if (g.e.bsum) {
    cudaError_t e;
    {
      ProfScope ps(c, "dcn.dT_fused", 2.0 * (double)g.M * g.N * g.K * g.batch, gemm_bytes(g) - overlap, st);
      e = gemm_run(g, c->ws, st);
      if (ps.rec >= 0) c->recs[ps.rec].tc = g_last_gemm_tc;
    }
    if (e == cudaSuccess) { *rows = g_last_gemm_grid; return DHEN_OK; }
    if (e != cudaErrorNotSupported) CK(e);
    (void)cudaGetLastError();
    g.e.bsum = nullptr;
  }
  ProfScope ps(c, "dcn.dT_fused", 2.0 * (double)g.M * g.N * g.K * g.batch, gemm_bytes(g) - overlap, st);
  CK(gemm_run(g, c->ws, st));
  if (ps.rec >= 0) c->recs[ps.rec].tc = g_last_gemm_tc;
  return DHEN_OK;
}
// A GEMM with fused column sums of its stored output (Epilogue::csum) when its TMA-store pass can take
// them; otherwise the same GEMM without (*ok = false: the caller sums the output itself).
static dhen_status G_csum(Gemm& g, dhen_ctx* c, cudaStream_t st, const char* tag, bool* ok) {
  *ok = false;
  if (g.e.csum) {
    cudaError_t e;
    {
      ProfScope ps(c, tag, 2.0 * (double)g.M * g.N * g.K * g.batch, gemm_bytes(g), st);
      e = gemm_run(g, c->ws, st);
      if (ps.rec >= 0) c->recs[ps.rec].tc = g_last_gemm_tc;
    }
    if (e == cudaSuccess) { *ok = true; return DHEN_OK; }
    if (e != cudaErrorNotSupported) CK(e);
    (void)cudaGetLastError();
    g.e.csum = nullptr;
  }
  return G_(g, c, st, tag);
}
static Gemm mk(int M, int N, int K, int batch, Operand a, Operand b, View cv) {
  Gemm g;
  g.M = M; g.N = N; g.K = K; g.batch = batch; g.a = a; g.b = b; g.c = cv;
  return g;
}

// Parameter pointers for the current layer group
struct PP {
  char* base;
  int es;
  void* operator()(int64_t off) const { return base + off * es; }
};

// Token projection (F10): U_b = W^T T_b, as ONE GEMM over rows r = (b, c) (M = B*d, two-level row
// index), N = l, K = m:  U[b,t,c] = sum_i T[b,i,c] W[i,t].  T_b is read MN-major (c contiguous) and
// the output is column-contiguous (lanes along rows in the epilogue).
static dhen_status tokmix_fwd(dhen_ctx* c, const void* T, int m, const void* W, int l, float* dst, int64_t ldb, int B,
                              int acc, cudaStream_t st) {
  const int d = c->d, dt = c->dt;
  Gemm g = mk(B * d, l, m, 1, operand2(T, dt, d, (int64_t)m * d, 1, d), operand(W, dt, 1, l),
              view2(dst, F32, d, ldb, 1, d));
  g.e.accumulate = acc;
  return G_(g, c, st, "tokmix.fwd");
}
// B4: dT[b,i,c] = sum_t W[i,t] dU[b,t,c] (rows (b,c), N = m, K = l) stored (dT_dt) or accumulated
// into fp32; dW[i,t] += sum_(b,c) T[b,i,c] dU[b,t,c] (K = B*d, two-level K).
// ... dgrad on `st`, wgrad on `sw` with workspace `wsw` (the weight-gradient side stream, or st itself)
static dhen_status tokmix_bwd(dhen_ctx* c, const void* T, int m, const void* W, int l, const void* dU, int64_t ldu,
                              void* dT, int dT_dt, int acc, float* gW, int B, cudaStream_t st, cudaStream_t sw = nullptr,
                              const Workspace* wsw = nullptr, const void* resid = nullptr, int resid_dt = -1) {
  const int d = c->d, dt = c->dt;
  // per-sample batched: dT_b = W dU_b (M = m rows i, N = d, K = l), row-major output; with `resid` (the
  // identity shortcut's dR, same [B][m][d] layout) it is the first writer: dT = resid + W dU_b
  Gemm g = mk(m, d, l, B, operand(W, dt, l, 1), operand(dU, dt, 1, d, ldu), view(dT, dT_dt, d, 1, (int64_t)m * d));
  g.e.accumulate = resid ? 0 : acc;
  if (resid) g.e.resid = view((void*)resid, resid_dt >= 0 ? resid_dt : dt, d, 1, (int64_t)m * d);
  RET(G_(g, c, st, "tokmix.dgrad"));
  Gemm gw = mk(m, l, B * d, 1, operand(T, dt, d, 1, 0, 0, 1, d, (int64_t)m * d),
               operand(dU, dt, d, 1, 0, 0, 1, d, ldu), view(gW, F32, l, 1));
  gw.e.accumulate = 1;
  return G_(gw, c, sw ? sw : st, "tokmix.wgrad", wsw);
}

// ------------------------------------------------------------------ FSDP gather / scatter
// Two gathered-parameter slots (slot = group & 1).  All collectives run on the communication stream:
//   prefetch(g): comm waits ev_use[slot] (the compute stream is done with the slot's previous owner),
//                all-gathers group g into the slot, records ev_ag[slot];
//   comp_params(g): prefetch if needed, then the compute stream waits ev_ag[slot];
//   release(g):  the compute stream records ev_use[slot] after the last kernel reading the slot;
//   reduce_grads(g): comm waits ev_grad (recorded on compute after g's backward), reduce-scatters the
//                fp32 gradient into the local shard (all-reduce in replicated DP mode).
// world == 1: parameters are local, nothing is launched.
static bool sharded(const dhen_ctx* c) { return c->dist.world > 1 && c->dist.fsdp; }

static dhen_status prefetch(dhen_ctx* c, int gi) {
  if (!sharded(c) || gi < 0 || gi > c->cfg.n_layers) return DHEN_OK;
  const int slot = gi & 1;
  if (c->gathered_owner[slot] == gi) return DHEN_OK;
  Group& g = c->G[gi];
  CK(cudaStreamWaitEvent(c->comm_st, c->ev_use[slot], 0));
  if (c->comm->all_gather(g.comp, c->gathered[slot], (size_t)g.shard, c->dt, c->comm_st))
    return fail(DHEN_E_NCCL, "all-gather of group %d (%s): %s", gi, c->comm->name(), c->comm->err.c_str());
  CK(cudaEventRecord(c->ev_ag[slot], c->comm_st));
  c->gathered_owner[slot] = gi;
  return DHEN_OK;
}
static dhen_status comp_params(dhen_ctx* c, int gi, cudaStream_t st, void** out) {
  Group& g = c->G[gi];
  if (!sharded(c)) { *out = g.comp; return DHEN_OK; }
  RET(prefetch(c, gi));
  CK(cudaStreamWaitEvent(st, c->ev_ag[gi & 1], 0));
  *out = c->gathered[gi & 1];
  return DHEN_OK;
}
static dhen_status release(dhen_ctx* c, int gi, cudaStream_t st) {
  if (!sharded(c)) return DHEN_OK;
  CK(cudaEventRecord(c->ev_use[gi & 1], st));
  return DHEN_OK;
}
static void invalidate_gathered(dhen_ctx* c) { c->gathered_owner[0] = c->gathered_owner[1] = -1; }
// parameters (compute copies) were rewritten on `st`: later all-gathers must wait for that
static dhen_status fence_params(dhen_ctx* c, cudaStream_t st) {
  invalidate_gathered(c);
  if (!sharded(c)) return DHEN_OK;
  for (int k = 0; k < 2; ++k) CK(cudaEventRecord(c->ev_use[k], st));
  return DHEN_OK;
}

// (`also`: a second stream whose pending work also produces this group's gradients, e.g. trailing head sums)
static dhen_status reduce_grads(dhen_ctx* c, int gi, cudaStream_t st, cudaStream_t also = nullptr) {
  if (c->dist.world == 1) return DHEN_OK;
  Group& g = c->G[gi];
  CK(cudaEventRecord(c->ev_grad, st));
  CK(cudaStreamWaitEvent(c->comm_st, c->ev_grad, 0));
  if (also && also != st) {
    CK(cudaEventRecord(c->ev_grad2, also));
    CK(cudaStreamWaitEvent(c->comm_st, c->ev_grad2, 0));
  }
  if (c->dist.grad_bf16) {
    // quantized gradient collective: the compute stream casts the fp32 gradient into one of two
    // bf16 buffers (after the reduction that last read it), the communication stream reduces in bf16 and
    // widens its shard into the fp32 gradient shard
    const int k = gi & 1;
    if (also && also != st) CK(cudaStreamWaitEvent(st, c->ev_grad2, 0));   // (trailing gradient sums)
    CK(cudaStreamWaitEvent(st, c->ev_rs[k], 0));
    KT("comm.grad_cast", 0, (double)g.npad * 6, cast(g.grad, F32, c->gbf[k], BF16, g.npad, st));
    CK(cudaEventRecord(c->ev_grad, st));
    CK(cudaStreamWaitEvent(c->comm_st, c->ev_grad, 0));
    const size_t n = c->dist.fsdp ? (size_t)g.shard : (size_t)g.npad;
    const int r = c->dist.fsdp ? c->comm->reduce_scatter(c->gbf[k], c->gbf_shard, n, BF16, c->comm_st)
                               : c->comm->all_reduce(c->gbf[k], c->gbf_shard, n, BF16, c->comm_st);
    if (r) return fail(DHEN_E_NCCL, "gradient reduction of group %d (%s): %s", gi, c->comm->name(), c->comm->err.c_str());
    CK(cudaEventRecord(c->ev_rs[k], c->comm_st));
    CK(cast(c->gbf_shard, BF16, g.gshard, F32, (int64_t)n, c->comm_st));
    return DHEN_OK;
  }
  const int r = c->dist.fsdp ? c->comm->reduce_scatter(g.grad, g.gshard, (size_t)g.shard, F32, c->comm_st)
                             : c->comm->all_reduce(g.grad, g.gshard, (size_t)g.shard, F32, c->comm_st);
  if (r) return fail(DHEN_E_NCCL, "gradient reduction of group %d (%s): %s", gi, c->comm->name(), c->comm->err.c_str());
  return DHEN_OK;
}
// the compute stream waits for every collective issued so far
static dhen_status join_comm(dhen_ctx* c, cudaStream_t st) {
  if (c->dist.world == 1) return DHEN_OK;
  CK(cudaEventRecord(c->ev_comm, c->comm_st));
  CK(cudaStreamWaitEvent(st, c->ev_comm, 0));
  return DHEN_OK;
}

// Whether layer n's forward takes the LayerNorm-fused form (F12 in the producing GEMMs' epilogues).
static bool layer_lnf(const dhen_ctx* c, int n, int B) {
  const Layer& Lr = c->L[n];
  const int d = c->d, mi = Lr.m_in, mo = Lr.m_out;
  bool lnf = c->tune.ln_fuse && c->dt == BF16 && Lr.Wn < 0 && mi == mo && (d == 128 || d == 256) && Lr.ens == DHEN_CONCAT &&
             !Lr.inj;   // (injection: the modules read the widened input, the LayerNorm the layer's own)
  for (const Mod& m_ : Lr.mods) lnf = lnf && m_.s.kind != DHEN_DCN_LIT;   // (its output goes through the fp32 concat)
  for (const Mod& m_ : Lr.mods) {
    if (!lnf) break;
    const int l_ = m_.s.l;
    if (m_.s.kind == DHEN_DOT || m_.s.kind == DHEN_MLP) {
      const int N = l_ * d, BN = N <= 64 ? 64 : N <= 128 ? 128 : 256;
      lnf = BN >= 128 && N % BN == 0 && (d == BN || 2 * d == BN);
    } else {
      lnf = l_ <= 128 && 128 % l_ == 0 && B % (128 / l_) == 0 && mi % 64 == 0 && (128 / l_) * mi <= 1024;
    }
  }
  return lnf;
}
// Whether the DCN backward's token-map dgrad packs 128 / m samples per tile (block-diagonal W_u).
static bool dcn_pack(const dhen_ctx* c, int mi, int l, int B) {
  const int spt = 128 / std::max(mi, 1);
  return c->dt == BF16 && mi <= 64 && 128 % mi == 0 && l <= 64 && 64 % l == 0 &&
         (spt * l) % 64 == 0 && B % spt == 0;
}

// ------------------------------------------------------------------ layer forward
static dhen_status layer_fwd(dhen_ctx* c, int n, const void* X, void* Y, int B, cudaStream_t st) {
  Layer& Lr = c->L[n];
  const int d = c->d, dt = c->dt, es = c->es;
  const int mi = Lr.m_mod, mo = Lr.m_out;   // (mi: the tokens the modules read; the shortcut reads Lr.m_in)
  void* pbase;
  RET(comp_params(c, n, st, &pbase));
  if (n == 0) c->x0_cur = X;
  const void* Xs = X;   // the shortcut's input X_n
  if (Lr.inj) {         // R38: the modules read [X_n ; D], D = X0's first dense_tokens tokens
    if (!c->x0_cur) return fail(DHEN_E_STATE, "layer %d injects dense tokens: layer 0's forward has not run", n);
    KT("layer.inject", 0, (double)B * (Lr.m_in + 2.0 * c->cfg.dense_tokens + mi) * d * es,
       inject_copy(Xs, c->x0_cur, dt, B, Lr.m_in, c->cfg.dense_tokens, c->cfg.m0, d, Lr.Xin, st));
    X = Lr.Xin;
  }
  PP p{(char*)pbase, es};
  float* U = c->Ucat;
  const int64_t ldU = (int64_t)mo * d;
  const int64_t rows = (int64_t)B * mi;
  // Module branches are independent until the concat (each writes its own token rows of Ucat): with a
  // self-attention module in the layer it runs on the layer stream and every other module on the side
  // stream; otherwise modules alternate.  Attention modules always stay on the layer stream (rtmp/big
  // scratch).  The profiled pass runs serialised.
  // F12 fused (identity shortcut, bf16, d = 128 / 256): every module's producing GEMM writes its token rows of
  // Y = LN(U_i + X) directly -- the LayerNorm runs in its epilogue over d-column segments (R, mu, rstd saved),
  // so neither the fp32 concat buffer nor the LayerNorm kernel is touched.  Token-mixing outputs use the packed
  // form U[(b, t)] = blockdiag(W_u^T, ..) x [T_b; T_b+1; ..] (rows = tokens of 128 / l samples per tile).
  const bool lnf = layer_lnf(c, n, B);
  const cudaStream_t st0 = st;
  const bool use_side = c->tune.overlap && !serial_prof(c) && Lr.mods.size() > 1;
  bool has_attn = false;
  for (const Mod& m_ : Lr.mods) has_attn |= m_.s.kind == DHEN_ATTN;
  if (use_side) { CK(cudaEventRecord(c->ev_sf, st0)); CK(cudaStreamWaitEvent(c->side_st, c->ev_sf, 0)); }
  int mod_idx = 0;
  for (Mod& md : Lr.mods) {
    const int l = md.s.l;
    // (sum / weighted-sum ensembles: each module writes its own fp32 output, combined with the LayerNorm below)
    float* Us = Lr.ens != DHEN_CONCAT ? md.Uo : U + (int64_t)md.off_tok * d;
    const bool on_side = use_side && md.s.kind != DHEN_ATTN && (has_attn || (mod_idx & 1));
    ++mod_idx;
    cudaStream_t st = on_side ? c->side_st : st0;   // this module's stream (shadows the layer stream)
    const int64_t so = (int64_t)mo * d;               // sample stride of Y / R / X (mi == mo when lnf)
    char* Yo = (char*)Y + (int64_t)md.off_tok * d * es;
    char* Ro = (char*)Lr.R + (int64_t)md.off_tok * d * es;
    const char* Xo = (const char*)X + (int64_t)md.off_tok * d * es;
    auto set_ln = [&](Gemm& gm) {
      gm.e.ln_gamma = p(Lr.gamma); gm.e.ln_beta = p(Lr.beta);
      gm.e.ln_mu = Lr.mu + md.off_tok; gm.e.ln_rstd = Lr.rstd + md.off_tok;
      gm.e.ln_eps = c->cfg.ln_eps; gm.e.ln_d = d;
    };
    // token projection U = W^T T of this module: into the concat buffer, or packed with the layer LN fused
    auto emit_tm = [&](const void* T_, const void* W_) -> dhen_status {
      if (!lnf) return tokmix_fwd(c, T_, mi, W_, l, Us, ldU, B, 0, st);
      const int spt = 128 / l;
      if (!md.bdT_pre) KT("tokmix.bdiagT", 0, 0.0, blockdiag_t(W_, mi, l, spt, md.bdT, st));
      auto rows2 = [&](void* ptr) { View v = view2(ptr, dt, l, so, d, 1); v.bs0 = spt * so; return v; };
      Gemm gm = mk(spt * l, d, spt * mi, B / spt, operand(md.bdT, dt, spt * mi, 1),
                   operand(T_, dt, 1, d, (int64_t)spt * mi * d, 0, 1, mi, (int64_t)mi * d), rows2(Yo));
      gm.e.resid = rows2((void*)Xo);
      gm.e.aux = rows2(Ro);
      set_ln(gm);
      return G_(gm, c, st, "tokmix.fwd_ln");
    };
    switch (md.s.kind) {
      case DHEN_DOT: {   // F1 + F2
        const int h = mi * (mi - 1) / 2;
        // Gram X X^T per sample; the epilogue writes the strict upper triangle Z directly (F1, R7)
        Gemm g = mk(mi, mi, d, B, operand(X, dt, d, 1, (int64_t)mi * d), operand(X, dt, d, 1, (int64_t)mi * d),
                    view(md.Z, dt, 0, 1, (int64_t)h));
        g.e.triu_m = mi;
        RET(G_(g, c, st, "dot.gram"));
        if (lnf) {   // F2 + F12: the projection's rows are samples, its columns l tokens x d (LN per d segment)
          Gemm v = mk(B, l * d, h, 1, operand(md.Z, dt, h, 1), operand(p(md.Wm), dt, h, 1), view(Yo, dt, so, 1));
          v.e.resid = view((void*)Xo, dt, so, 1);
          v.e.aux = view(Ro, dt, so, 1);
          set_ln(v);
          RET(G_(v, c, st, "dot.proj_ln"));
        } else {
          Gemm v = mk(B, l * d, h, 1, operand(md.Z, dt, h, 1), operand(p(md.Wm), dt, h, 1), view(Us, F32, ldU, 1));
          RET(G_(v, c, st, "dot.proj"));
        }
        break;
      }
      case DHEN_LINEAR:  // F10 with T = X
        RET(emit_tm(X, p(md.W)));
        break;
      case DHEN_DCN: case DHEN_DCN_FULL: {   // F8: A = X W^T + b ; T = X * A + X (per token, or R37 per sample)
        const bool flat = md.s.kind == DHEN_DCN_FULL;
        const int w = flat ? mi * d : d;
        Gemm g = mk(flat ? B : (int)rows, w, w, 1, operand(X, dt, w, 1), operand(p(md.W), dt, w, 1), view(md.T, dt, w, 1));
        g.e.bias = p(md.b); g.e.bias_dt = dt;
        g.e.cross = view((void*)X, dt, w, 1);
        g.e.aux = view(md.A, dt, w, 1);
        RET(G_(g, c, st, "dcn.cross"));
        RET(emit_tm(md.T, p(md.Wu)));
        break;
      }
      case DHEN_CONV:    // F7
        KT("conv.fwd", 2.0 * rows * d * md.s.conv_k * md.s.conv_k, 2.0 * rows * d * es, conv_fwd(X, p(md.K), dt, md.s.conv_channels, md.s.conv_k, B, mi, d, md.T, dt, st));
        RET(emit_tm(md.T, p(md.Wu)));
        break;
      case DHEN_ATTN: {  // F3-F6
        const int H = md.s.heads, dh = d / H, f = md.s.ffn_mult * d;
        const int64_t s3 = 3 * (int64_t)d;
        char* QKV = (char*)md.QKV;
        Gemm q = mk((int)rows, 3 * d, d, 1, operand(X, dt, d, 1), operand(p(md.Wq), dt, d, 1), view(QKV, dt, s3, 1));
        q.e.bias = p(md.bq); q.e.bias_dt = dt; q.e.bias_gap_lo = d; q.e.bias_gap_hi = 2 * d;   // no key bias (R10)
        q.e.bias_hi_off = (int)(md.bv - md.bq);
        RET(G_(q, c, st, "attn.qkv"));
        if (attn::fused_ok(dt, B, H, mi, d)) {
          // F4 fused: S, softmax and P V per (sample, head) on one SM, P never leaves shared memory
          ProfScope ps(c, "attn.core", 4.0 * B * H * (double)mi * mi * dh, (double)B * mi * 4 * d * es, st);
          CK(attn::core_fwd(QKV, md.O, B, H, mi, d, st));
          if (ps.rec >= 0) c->recs[ps.rec].tc = 1;
        } else {
          const int mp = (mi + 7) / 8 * 8;   // padded score-row pitch
          Gemm s = mk(mi, mi, dh, B * H, operand(QKV, dt, s3, 1, mi * s3, dh, H),
                      operand(QKV + (int64_t)d * es, dt, s3, 1, mi * s3, dh, H),
                      view(c->big, F32, mp, 1, (int64_t)mi * mp));
          s.e.alpha = 1.f / sqrtf((float)dh);
          RET(G_(s, c, st, "attn.qk"));
          KT("attn.softmax", 0, (double)B * H * mi * mi * (4 + es), softmax_rows(c->big, md.P, dt, (int64_t)B * H * mi, mi, mp, st));
          Gemm o = mk(mi, dh, mi, B * H, operand(md.P, dt, mp, 1, (int64_t)mi * mp),
                      operand(QKV + 2 * (int64_t)d * es, dt, 1, s3, mi * s3, dh, H),
                      view(md.O, dt, d, 1, (int64_t)mi * d, dh, H));
          RET(G_(o, c, st, "attn.pv"));
        }
        // F5: Z1 = LN1(X + O W_o^T + b_o) -- with whole rows per tile (bf16, d = 128 / 256) the LayerNorm runs
        // in the GEMM epilogue (R1 and the row statistics saved for B6), else GEMM into fp32 + LN kernel
        const bool ln_fused = c->tune.ln_fuse && dt == BF16 && (d == 128 || d == 256);
        if (ln_fused) {
          Gemm r1 = mk((int)rows, d, d, 1, operand(md.O, dt, d, 1), operand(p(md.Wo), dt, d, 1), view(md.Z1, dt, d, 1));
          r1.e.bias = p(md.bo); r1.e.bias_dt = dt; r1.e.resid = view((void*)X, dt, d, 1);
          r1.e.aux = view(md.R1, dt, d, 1);
          r1.e.ln_gamma = p(md.g1); r1.e.ln_beta = p(md.be1); r1.e.ln_mu = md.mu1; r1.e.ln_rstd = md.rs1;
          r1.e.ln_eps = c->cfg.ln_eps;
          RET(G_(r1, c, st, "attn.out_ln1"));
        } else {
          Gemm r1 = mk((int)rows, d, d, 1, operand(md.O, dt, d, 1), operand(p(md.Wo), dt, d, 1), view(c->rtmp, F32, d, 1));
          r1.e.bias = p(md.bo); r1.e.bias_dt = dt; r1.e.resid = view((void*)X, dt, d, 1);
          RET(G_(r1, c, st, "attn.out"));
          KT("attn.ln1", 0, (double)rows * d * (4 + 2 * es), ln_fwd(c->rtmp, nullptr, p(md.g1), p(md.be1), dt, c->cfg.ln_eps, rows, d, md.Z1, md.R1, md.mu1, md.rs1, dt, st));
        }
        Gemm f1 = mk((int)rows, f, d, 1, operand(md.Z1, dt, d, 1), operand(p(md.W1), dt, d, 1), view(md.F, dt, f, 1));
        f1.e.bias = p(md.b1); f1.e.bias_dt = dt; f1.e.relu = 1;
        // (the bitmask is written / read by the TMA-store epilogue only)
        const bool fbits = c->tune.relu_bits && c->tune.tstore && dt == BF16 && f % 64 == 0 && f >= 128;
        if (fbits) { f1.e.bits = md.Fbits; f1.e.bits_mode = 1; f1.e.bits_ld = rows; }
        RET(G_(f1, c, st, "attn.ffn1"));
        // F6: T = LN2(Z1 + F W_2^T + b_2), fused the same way
        if (ln_fused) {
          Gemm f2 = mk((int)rows, d, f, 1, operand(md.F, dt, f, 1), operand(p(md.W2), dt, f, 1), view(md.T, dt, d, 1));
          f2.e.bias = p(md.b2); f2.e.bias_dt = dt; f2.e.resid = view(md.Z1, dt, d, 1);
          f2.e.aux = view(md.R2, dt, d, 1);
          f2.e.ln_gamma = p(md.g2); f2.e.ln_beta = p(md.be2); f2.e.ln_mu = md.mu2; f2.e.ln_rstd = md.rs2;
          f2.e.ln_eps = c->cfg.ln_eps;
          RET(G_(f2, c, st, "attn.ffn2_ln2"));
        } else {
          Gemm f2 = mk((int)rows, d, f, 1, operand(md.F, dt, f, 1), operand(p(md.W2), dt, f, 1), view(c->rtmp, F32, d, 1));
          f2.e.bias = p(md.b2); f2.e.bias_dt = dt; f2.e.resid = view(md.Z1, dt, d, 1);
          RET(G_(f2, c, st, "attn.ffn2"));
          KT("attn.ln2", 0, (double)rows * d * (4 + 2 * es), ln_fwd(c->rtmp, nullptr, p(md.g2), p(md.be2), dt, c->cfg.ln_eps, rows, d, md.T, md.R2, md.mu2, md.rs2, dt, st));
        }
        RET(emit_tm(md.T, p(md.Wu)));
        break;
      }
      case DHEN_DCN_LIT: {   // Eq.(7) literally (R31): G_b = X_b^T X_b (d x d), U_b = W^T G_b + b
        Gemm g = mk(d, d, mi, B, operand(X, dt, 1, d, (int64_t)mi * d), operand(X, dt, 1, d, (int64_t)mi * d),
                    view(md.G, dt, d, 1, (int64_t)d * d));
        RET(G_(g, c, st, "dcnl.gram"));
        Gemm u = mk(l, d, d, B, operand(p(md.W), dt, 1, l), operand(md.G, dt, 1, d, (int64_t)d * d),
                    view(Us, F32, d, 1, ldU));
        u.e.resid = view(p(md.b), dt, d, 1, 0);   // the [l][d] bias, the same for every sample
        RET(G_(u, c, st, "dcnl.proj"));
        break;
      }
      case DHEN_MLP: {   // F9
        const int h1 = md.s.mlp_hidden[0], h2 = md.s.mlp_hidden[1];
        const int K1 = mi * d;
        Gemm a = mk(B, h1, K1, 1, operand(X, dt, K1, 1), operand(p(md.W1), dt, K1, 1), view(md.h1, dt, h1, 1));
        a.e.bias = p(md.b1); a.e.bias_dt = dt; a.e.relu = 1;
        RET(G_(a, c, st, "mlp.fc1"));
        Gemm b2 = mk(B, h2, h1, 1, operand(md.h1, dt, h1, 1), operand(p(md.W2), dt, h1, 1), view(md.h2, dt, h2, 1));
        b2.e.bias = p(md.b2); b2.e.bias_dt = dt; b2.e.relu = 1;
        RET(G_(b2, c, st, "mlp.fc2"));
        if (lnf) {
          Gemm v = mk(B, l * d, h2, 1, operand(md.h2, dt, h2, 1), operand(p(md.Wm), dt, h2, 1), view(Yo, dt, so, 1));
          v.e.resid = view((void*)Xo, dt, so, 1);
          v.e.aux = view(Ro, dt, so, 1);
          set_ln(v);
          RET(G_(v, c, st, "mlp.proj_ln"));
        } else {
          Gemm v = mk(B, l * d, h2, 1, operand(md.h2, dt, h2, 1), operand(p(md.Wm), dt, h2, 1), view(Us, F32, ldU, 1));
          RET(G_(v, c, st, "mlp.proj"));
        }
        break;
      }
    }
  }
  if (use_side) { CK(cudaEventRecord(c->ev_sj, c->side_st)); CK(cudaStreamWaitEvent(st0, c->ev_sj, 0)); }
  // F11 shortcut (Eq.(2)) + F12 LayerNorm
  if (Lr.Wn >= 0) RET(tokmix_fwd(c, Xs, Lr.m_in, p(Lr.Wn), mo, U, ldU, B, Lr.ens == DHEN_CONCAT ? 1 : 0, st));
  if (Lr.ens != DHEN_CONCAT) {   // R = sum_i (w_i) U_i + shortcut, then the layer LayerNorm (R27)
    EnsU eu;
    eu.k = (int)Lr.mods.size();
    for (int i = 0; i < eu.k; ++i) eu.u[i] = Lr.mods[i].Uo;
    KT("layer.ens_ln", 0, (double)B * mo * d * (4.0 * eu.k + 2 * es + es),
       ens_ln_fwd(eu, Lr.ens == DHEN_WSUM ? p(Lr.ensw) : nullptr, dt, Lr.Wn >= 0 ? U : nullptr, Lr.Wn >= 0 ? nullptr : Xs,
                  p(Lr.gamma), p(Lr.beta), c->cfg.ln_eps, (int64_t)B * mo, d, Y, Lr.R, Lr.mu, Lr.rstd, dt, st));
  } else if (!lnf)
    KT("layer.ln", 0, (double)B * mo * d * (4 + 2 * es) + (Lr.Wn >= 0 ? 0.0 : (double)B * mo * d * es), ln_fwd(U, Lr.Wn >= 0 ? nullptr : Xs, p(Lr.gamma), p(Lr.beta), dt, c->cfg.ln_eps, (int64_t)B * mo, d, Y, Lr.R, Lr.mu,
              Lr.rstd, dt, st));
  Lr.X = X;     // the modules' input
  Lr.Xs = Xs;   // the shortcut's
  Lr.B = B;
  RET(release(c, n, st));
  return DHEN_OK;
}

// ------------------------------------------------------------------ layer backward
static dhen_status layer_bwd(dhen_ctx* c, int n, const void* dY, void* dX, int B, cudaStream_t st) {
  Layer& Lr = c->L[n];
  Group& G = c->G[n];
  const int d = c->d, dt = c->dt, es = c->es;
  const int mi = Lr.m_mod, mo = Lr.m_out;   // (mi: the tokens the modules read, R38)
  const void* X = Lr.X;
  void* pbase;
  RET(comp_params(c, n, st, &pbase));
  PP p{(char*)pbase, es};
  float* g = G.grad;
  auto gp = [&](int64_t off) { return g + off; };
  const int64_t ldU = (int64_t)mo * d;
  const int64_t rows = (int64_t)B * mi;
  // R38 route (an injected layer, or layer 0 when any layer injects): the modules accumulate into their own
  // [B][m_mod][d] buffer; the shortcut's part stays in dXacc; a final kernel forms dX (+ dD at layer 0)
  const bool route = Lr.inj || (n == 0 && c->dense_active);
  if (c->dense_active && n == c->cfg.n_layers - 1)   // the first backward layer of the step: dD starts at 0
    CK(cudaMemsetAsync(c->dD, 0, (size_t)B * c->cfg.dense_tokens * d * 4, st));
  float* acc_sc = c->dXacc;
  float* acc = route ? c->dXacc2 : acc_sc;
  if (route) CK(cudaMemsetAsync(acc, 0, (size_t)B * mi * d * 4, st));
  // B2: LN backward; identity shortcut (B3) initialises the dX accumulator
  // B3 identity shortcut: dX starts as dR.  When the first module's first dX-writing GEMM can add dR in its
  // epilogue (Dot: Gram backward, DCN: dT, Linear: token dgrad, MLP: fc1 dgrad) it initialises the fp32
  // accumulator itself and LN backward does not write it (one fp32 write + one read-modify-write saved).
  // Module order of the backward: the best first-writer candidate goes first (its epilogue adds dR most
  // cheaply: DCN > Linear > MLP > Dot), the others follow in declaration order (a fixed order: deterministic).
  std::vector<Mod*> order;
  {
    int best = -1, best_rank = 99;
    const int rank_of[8] = {3 /*DOT*/, 99 /*ATTN*/, 99 /*CONV*/, 0 /*DCN*/, 1 /*LINEAR*/, 2 /*MLP*/, 99 /*DCN_LIT*/,
                            0 /*DCN_FULL*/};
    for (int i = 0; i < (int)Lr.mods.size(); ++i) {
      const int rk = rank_of[Lr.mods[i].s.kind];
      if (rk < best_rank) { best_rank = rk; best = i; }
    }
    if (best >= 0 && c->tune.first_writer) order.push_back(&Lr.mods[best]);
    for (int i = 0; i < (int)Lr.mods.size(); ++i)
      if (!(c->tune.first_writer && i == best)) order.push_back(&Lr.mods[i]);
  }
  const int first_kind = order.empty() ? -1 : order[0]->s.kind;
  const bool first_dR = c->tune.first_writer && !route && Lr.Wn < 0 && mi == mo &&
                        (first_kind == DHEN_DOT || first_kind == DHEN_DCN || first_kind == DHEN_DCN_FULL ||
                         first_kind == DHEN_LINEAR || first_kind == DHEN_MLP);
  // Weight gradients of a module run on the side stream `sd` (own split-K / reduction scratch) while its
  // data gradients run on `st`; `fork` hands the side stream everything enqueued on st so far, and st waits
  // for the side stream before it overwrites a shared buffer that pending side work reads (and at layer end).
  // (the profiled pass runs serialised so every op's event-timed duration is its own)
  cudaStream_t sd = (c->tune.overlap && !serial_prof(c)) ? c->side_st : st;
  // the LN parameter sums trail on sd (own scratch red3; the modules' joins below order its reuse)
  KT("layer.ln_bwd", 0, (double)B * mo * d * (3 * es + (first_dR ? 0 : 4)), ln_bwd(dY, dt, Lr.R, Lr.mu, Lr.rstd, p(Lr.gamma), dt, (int64_t)B * mo, d, c->dR, dt, acc_sc, (Lr.Wn >= 0 || first_dR) ? 0 : 1,
            gp(Lr.gamma), gp(Lr.beta), c->red3, c->red_bytes, st, c->tune.trail ? sd : st, c->ev_red,
            c->vdy_now ? c->dz : nullptr, c->vdy_now ? (sharded(c) ? c->headw : c->G[c->cfg.n_layers].comp) : nullptr, mo));
  c->vdy_now = false;
  if (Lr.Wn >= 0)   // B3: dX = W_n dR ; dW_n += sum_b X_b dR_b^T
    RET(tokmix_bwd(c, Lr.Xs, Lr.m_in, p(Lr.Wn), mo, c->dR, ldU, acc_sc, F32, 0, gp(Lr.Wn), B, st));
  const Workspace* ws2 = &c->ws2;
  float* red2 = c->red2;
  auto fork = [&]() -> dhen_status {
    if (sd != st) { CK(cudaEventRecord(c->ev_sf, st)); CK(cudaStreamWaitEvent(sd, c->ev_sf, 0)); }
    return DHEN_OK;
  };
  // Joins are deferred: a module's side-stream work only has to finish before later st work overwrites a
  // shared buffer it reads.  Bits: 1 tA, 2 tB, 4 tC, 8 tD, 16 bsum, 32 tE, 64 tF, 128 rtmp, 256 big, 512 csum.
  // (Conv and MLP backward scratch is per module, so they share nothing.)
  auto st_writes = [](int k) -> uint32_t {
    switch (k) {
      case DHEN_DOT: return 1u | 8u;      // dZ (tA), S (tD)
      case DHEN_DCN: case DHEN_DCN_FULL: return 2u | 16u;     // dA (tB), dA column sums (bsum)
      case DHEN_ATTN: return 1u | 2u | 4u | 8u | 32u | 64u | 128u | 256u | 512u | 1024u;   // (1024: F, when shared)
      case DHEN_CONV: case DHEN_MLP: case DHEN_LINEAR: case DHEN_DCN_LIT: return 0u;   // own scratch / the dX accumulator
      default: return ~0u;
    }
  };
  auto side_reads = [](int k) -> uint32_t {
    switch (k) {
      case DHEN_DCN: case DHEN_DCN_FULL: return 2u | 16u;     // dA, its column sums
      case DHEN_ATTN: return 1u | 2u | 4u | 64u | 512u | 1024u;   // dR2 (tA), dR1 (tB), dF (tC), dQKV (tF), db1, F
      case DHEN_DOT: case DHEN_CONV: case DHEN_MLP: case DHEN_LINEAR: case DHEN_DCN_LIT: return 0u;   // saved / own buffers
      default: return ~0u;
    }
  };
  uint32_t side_pending = 0;
  int cur_kind = -1;
  auto real_join = [&]() -> dhen_status {
    if (sd != st) { CK(cudaEventRecord(c->ev_sj, sd)); CK(cudaStreamWaitEvent(st, c->ev_sj, 0)); }
    side_pending = 0;
    return DHEN_OK;
  };
  auto join = [&]() -> dhen_status {   // end of a module: record what its side work still reads
    side_pending |= side_reads(cur_kind);
    return c->tune.defer_join ? DHEN_OK : real_join();
  };
  // The last module's last dX-writing GEMM emits dX (layer dtype) = accumulator + its contribution: the fp32
  // accumulator is read once and never written back, and no cast kernel runs.
  const int last_kind = order.empty() ? -1 : order.back()->s.kind;
  const bool last_dX = dX && c->tune.first_writer && !route &&
                       (last_kind == DHEN_DOT || last_kind == DHEN_DCN || last_kind == DHEN_DCN_FULL ||
                        last_kind == DHEN_LINEAR || last_kind == DHEN_MLP);
  bool first_mod = true;
  for (Mod* mdp : order) {
    Mod& md = *mdp;
    const int l = md.s.l;
    char* dU = (char*)c->dR + (int64_t)md.off_tok * d * es;   // (sum ensembles: off_tok = 0, dU_i = dR)
    if (Lr.ens == DHEN_WSUM) {   // dU_i = w_i dR;  dw_i += <U_i, dR>  (R27)
      const int mi_idx = (int)(mdp - Lr.mods.data());
      KT("layer.ens_bwd", 0, (double)rows * d * (2.0 * es),
         ens_scale(c->dR, p(Lr.ensw), mi_idx, dt, md.dUs, (int64_t)B * mo * d, dt, st));
      KT("layer.ens_bwd", 0, (double)B * mo * d * (4.0 + es),
         ens_dot(md.Uo, c->dR, dt, (int64_t)B * mo * d, gp(Lr.ensw) + mi_idx, c->red, st));
      dU = (char*)md.dUs;
    }
    const bool take_dR = first_dR && first_mod;   // this module's first dX write adds the shortcut's dR
    const bool emit_dX = last_dX && mdp == order.back();   // this module's last dX write emits dX
    first_mod = false;
    cur_kind = md.s.kind;
    if (side_pending & st_writes(cur_kind)) RET(real_join());
    switch (md.s.kind) {
      case DHEN_DOT: {   // B5
        const int h = mi * (mi - 1) / 2;
        RET(fork());
        Gemm gw = mk(l * d, h, B, 1, operand(dU, dt, 1, ldU), operand(md.Z, dt, 1, h), view(gp(md.Wm), F32, h, 1));
        gw.e.accumulate = 1;
        RET(G_(gw, c, sd, "dot.proj_wgrad", ws2));
        Gemm gz = mk(B, h, l * d, 1, operand(dU, dt, ldU, 1), operand(p(md.Wm), dt, 1, h), view(c->tA, dt, h, 1));
        RET(G_(gz, c, st, "dot.proj_dgrad"));
        // dX_b (+)= S_b X_b with S built on chip from the packed dZ (no dense S in HBM): one kernel
        // (m <= 64, two samples per tile: the dense-S path measured faster, C2 118 vs 122 us / step)
        if (c->tune.sym < 0 && dt == BF16 && mi > 64 && dotb::supported(B, mi, d, h)) {
          const int mode = (take_dR ? 1 : 0) + (emit_dX ? 2 : 0);
          const void* rin = take_dR ? (const void*)c->dR : emit_dX ? (const void*)acc : nullptr;
          void* out = emit_dX ? dX : (void*)acc;
          // algorithmic bytes: dZ + X in; dX out (fp32 +=: read + write; first writer: dR in + fp32 out; emit: fp32
          // acc or dR in + bf16 out)
          const double rows_d = (double)B * mi * d;
          const double io = mode == 0 ? 8.0 * rows_d : mode == 1 ? 6.0 * rows_d : mode == 2 ? 6.0 * rows_d : 4.0 * rows_d;
          ProfScope ps(c, "dot.gram_bwd", 2.0 * B * (double)mi * mi * d, (double)B * h * es + rows_d * es + io, st);
          CK(dotb::gram_bwd(c->tA, h, X, B, mi, d, mode, rin, out, st));
          if (ps.rec >= 0) c->recs[ps.rec].tc = 1;
          RET(join());
          break;
        }
        KT("dot.sym", 0, (double)B * (h + mi * mi) * es, sym_from_triu(c->tA, c->tD, dt, B, mi, h, st));
        // dX_b += S_b X_b
        Gemm gx = mk(mi, d, mi, B, operand(c->tD, dt, mi, 1, (int64_t)mi * mi), operand(X, dt, 1, d, (int64_t)mi * d),
                     view(acc, F32, d, 1, (int64_t)mi * d));
        gx.e.accumulate = 1;
        if (take_dR) { gx.e.accumulate = 0; gx.e.resid = gx.c; gx.e.resid.ptr = c->dR; gx.e.resid.dt = dt; }
        if (emit_dX) {   // dX = (dR | acc) + S X
          if (!take_dR) { gx.e.resid = gx.c; }   // fp32 accumulator view
          gx.e.accumulate = 0;
          gx.c.ptr = dX; gx.c.dt = dt;
        }
        RET(G_(gx, c, st, "dot.gram_bwd"));
        RET(join());
        break;
      }
      case DHEN_LINEAR:
        RET(fork());
        if (emit_dX)   // dX = (dR | acc) + W dU
          RET(tokmix_bwd(c, X, mi, p(md.W), l, dU, ldU, dX, dt, 0, gp(md.W), B, st, sd, ws2,
                         take_dR ? (const void*)c->dR : (const void*)acc, take_dR ? dt : F32));
        else
          RET(tokmix_bwd(c, X, mi, p(md.W), l, dU, ldU, acc, F32, 1, gp(md.W), B, st, sd, ws2, take_dR ? c->dR : nullptr));
        RET(join());
        break;
      case DHEN_DCN: case DHEN_DCN_FULL: {   // B8 (R37: the dA W and dW contractions over the flattened sample)
        const bool flat = md.s.kind == DHEN_DCN_FULL;
        const int wf = flat ? mi * d : d;            // width of the cross contraction
        const int64_t rf = flat ? B : rows;          // its rows
        void* dA = c->tB;
        RET(fork());
        {   // dW_u += sum T dU (side stream; needs only saved T and dU)
          Gemm gw_u = mk(mi, l, B * d, 1, operand(md.T, dt, d, 1, 0, 0, 1, d, (int64_t)mi * d),
                         operand(dU, dt, d, 1, 0, 0, 1, d, ldU), view(gp(md.Wu), F32, l, 1));
          gw_u.e.accumulate = 1;
          RET(G_(gw_u, c, sd, "tokmix.wgrad", ws2));
        }
        // dT = W_u dU (never stored): the epilogue forms dA = dT (.) X and dX += dT (.) A + dT (B8)
        // m <= 64 (dividing 128), l dividing 64: spt = 128 / m samples per 128-row tile, as one GEMM with the
        // block-diagonal token map blockdiag(W_u, .., W_u) [spt m][spt l] against spt stacked dU_b (the B
        // operand's two-level K: k -> (sample, t)), so every MMA row and epilogue warp carries data.
        const int spt = 128 / std::max(mi, 1);
        const bool pack = dcn_pack(c, mi, l, B);
        // the bias gradient's column sums of dA come out of the dT GEMM's epilogue (one partial row per CTA)
        const bool fuse_db = c->tune.fuse_db && dt == BF16 && d <= 256 && !flat;   // (flat: db has m d entries)
        int bsum_rows = 0;
        const double dU_in_dR = take_dR ? (double)B * l * d * es : 0.0;   // dU is a slice of the dR residual
        const bool fused_bwd = !flat && c->tune.dcn_fused && dt == BF16 && (mi == 128 || pack) &&
                               dcnb::supported(B, mi, l, d, ldU, take_dR ? 0 : 1, emit_dX ? 0 : 1);
        if (fused_bwd) {
          // one kernel: dT = W_u dU, dA = dT (.) X, dX = base + dT (.) A + dT + dA W (partial dX in TMEM)
          const void* wu = p(md.Wu);
          if (mi < 128) {   // several samples per tile: the block-diagonal token map
            void* bdg = md.bdg_pre ? md.bdg : c->bdiag;
            if (!md.bdg_pre) KT("dcn.bdiag", 0, 2.0 * 128 * 128 * es, blockdiag(p(md.Wu), mi, l, spt, bdg, st));
            wu = bdg;
          }
          const double rd = (double)rows * d;
          // algorithmic bytes: dU + X + A + base in, dA + dX out (W, W_u once)
          const double bytes = (double)B * l * d * es + rd * (es + es + (take_dR ? es : 4) + es + (emit_dX ? es : 4)) +
                               (double)d * d * es - dU_in_dR;
          ProfScope ps(c, "dcn.bwd_fused", 2.0 * rows * l * d + 2.0 * rd * d, bytes, st);
          CK(dcnb::bwd(wu, dU, ldU, p(md.W), X, md.A, take_dR ? (const void*)c->dR : (const void*)acc, take_dR ? 0 : 1,
                       emit_dX ? dX : (void*)acc, emit_dX ? 0 : 1, dA, fuse_db ? c->bsum : nullptr, B, mi, l, d, st,
                       &bsum_rows));
          if (ps.rec >= 0) c->recs[ps.rec].tc = 1;
        } else if (pack) {
          void* bdg = md.bdg_pre ? md.bdg : c->bdiag;
          if (!md.bdg_pre) KT("dcn.bdiag", 0, 2.0 * 128 * 128 * es, blockdiag(p(md.Wu), mi, l, spt, bdg, st));
          Gemm gt = mk(spt * mi, d, spt * l, B / spt, operand(bdg, dt, spt * l, 1),
                       operand(dU, dt, 1, d, spt * ldU, 0, 1, l, ldU), view(acc, F32, d, 1, (int64_t)spt * mi * d));
          gt.e.dcn_bwd = 1;
          gt.e.cross = view((void*)X, dt, d, 1, (int64_t)spt * mi * d);
          gt.e.mask = view(md.A, dt, d, 1, (int64_t)spt * mi * d);
          gt.e.aux = view(dA, dt, d, 1, (int64_t)spt * mi * d);
          if (take_dR) gt.e.resid = view(c->dR, dt, d, 1, (int64_t)spt * mi * d);
          if (fuse_db) gt.e.bsum = c->bsum;
            RET(G_dT(gt, c, st, &bsum_rows, dU_in_dR));
        } else {
          Gemm gt = mk(mi, d, l, B, operand(p(md.Wu), dt, l, 1), operand(dU, dt, 1, d, ldU),
                       view(acc, F32, d, 1, (int64_t)mi * d));
          gt.e.dcn_bwd = 1;
          gt.e.cross = view((void*)X, dt, d, 1, (int64_t)mi * d);
          gt.e.mask = view(md.A, dt, d, 1, (int64_t)mi * d);
          gt.e.aux = view(dA, dt, d, 1, (int64_t)mi * d);
          if (take_dR) gt.e.resid = view(c->dR, dt, d, 1, (int64_t)mi * d);
          if (fuse_db) gt.e.bsum = c->bsum;
        RET(G_dT(gt, c, st, &bsum_rows, dU_in_dR));
        }
        if (sd != st) { CK(cudaEventRecord(c->ev_sx, st)); CK(cudaStreamWaitEvent(sd, c->ev_sx, 0)); }   // dA ready
        if (!fused_bwd) {
          Gemm gx = mk((int)rf, wf, wf, 1, operand(dA, dt, wf, 1), operand(p(md.W), dt, 1, wf), view(acc, F32, wf, 1));
          gx.e.accumulate = 1;
          if (emit_dX) { gx.e.accumulate = 0; gx.e.resid = view(acc, F32, wf, 1); gx.c = view(dX, dt, wf, 1); }   // dX = acc + dA W
          RET(G_(gx, c, st, "dcn.dgrad"));
        }
        Gemm gw = mk(wf, wf, (int)rf, 1, operand(dA, dt, 1, wf), operand(X, dt, 1, wf), view(gp(md.W), F32, wf, 1));
        gw.e.accumulate = 1;
        RET(G_(gw, c, sd, "dcn.wgrad", ws2));
        if (bsum_rows > 0)
          KTS(sd, "dcn.bias_grad", 0, (double)bsum_rows * d * 4, rows_sum_add(c->bsum, bsum_rows, d, gp(md.b), sd));
        else
          KTS(sd, "dcn.bias_grad", 0, (double)rows * d * es, colsum_add(dA, dt, rf, wf, wf, gp(md.b), red2, c->red_bytes, sd));
        RET(join());
        break;
      }
      case DHEN_CONV: {  // B7
        void* dT = md.dT;
        RET(fork());
        RET(tokmix_bwd(c, md.T, mi, p(md.Wu), l, dU, ldU, dT, dt, 0, gp(md.Wu), B, st, sd, ws2));
        if (sd != st) { CK(cudaEventRecord(c->ev_sx, st)); CK(cudaStreamWaitEvent(sd, c->ev_sx, 0)); }   // dT ready
        KT("conv.dgrad", 2.0 * rows * d * md.s.conv_k * md.s.conv_k, (double)rows * d * (es + 8), conv_dgrad(dT, p(md.K), dt, md.s.conv_channels, md.s.conv_k, B, mi, d, acc, dt, st));
        KTS(sd, "conv.wgrad", 2.0 * rows * d * md.s.conv_k * md.s.conv_k, 2.0 * rows * d * es, conv_wgrad(dT, X, md.s.conv_channels, md.s.conv_k, B, mi, d, dt, gp(md.K), red2, c->red_bytes, sd));
        RET(join());
        break;
      }
      case DHEN_ATTN: {  // B6
        const int H = md.s.heads, dh = d / H, f = md.s.ffn_mult * d;
        const int64_t s3 = 3 * (int64_t)d;
        char* QKV = (char*)md.QKV;
        void* dT = c->tB;
        // weight gradients and bias column sums run on the side stream as their inputs become ready
        // (dO and dQKV have their own buffers, so nothing the side stream reads is overwritten)
        auto ready = [&]() -> dhen_status {
          if (sd != st) { CK(cudaEventRecord(c->ev_sx, st)); CK(cudaStreamWaitEvent(sd, c->ev_sx, 0)); }
          return DHEN_OK;
        };
        RET(fork());
        if (c->cfg.recompute & 1) {   // NEXT#2: F (and its ReLU bitmask) recomputed from the saved Z1, bit-identical
          Gemm f1 = mk((int)rows, f, d, 1, operand(md.Z1, dt, d, 1), operand(p(md.W1), dt, d, 1), view(md.F, dt, f, 1));
          f1.e.bias = p(md.b1); f1.e.bias_dt = dt; f1.e.relu = 1;
          if (c->tune.relu_bits && c->tune.tstore && dt == BF16 && f % 64 == 0 && f >= 128) {
            f1.e.bits = md.Fbits; f1.e.bits_mode = 1; f1.e.bits_ld = rows;
          }
          RET(G_(f1, c, st, "attn.ffn1_recompute"));
        }
        RET(tokmix_bwd(c, md.T, mi, p(md.Wu), l, dU, ldU, dT, dt, 0, gp(md.Wu), B, st, sd, ws2));
        void* dR2 = c->tA;   // [rows, d]
        KT("attn.ln2_bwd", 0, (double)rows * d * 3 * es, ln_bwd(dT, dt, md.R2, md.mu2, md.rs2, p(md.g2), dt, rows, d, dR2, dt, nullptr, 0, gp(md.g2), gp(md.be2), c->red,
                  c->red_bytes, st));
        RET(ready());   // dR2
        {
          Gemm w2 = mk(d, f, (int)rows, 1, operand(dR2, dt, 1, d), operand(md.F, dt, 1, f), view(gp(md.W2), F32, f, 1));
          w2.e.accumulate = 1;
          RET(G_(w2, c, sd, "attn.ffn2_wgrad", ws2));
          KTS(sd, "attn.bias_grad", 0, (double)rows * d * es, colsum_add(dR2, dt, rows, d, d, gp(md.b2), red2, c->red_bytes, sd));
        }
        void* dF = c->tC;
        Gemm a = mk((int)rows, f, d, 1, operand(dR2, dt, d, 1), operand(p(md.W2), dt, 1, f), view(dF, dt, f, 1));
        if (c->tune.relu_bits && c->tune.tstore && dt == BF16 && f % 64 == 0 && f >= 128) {   // ReLU'(0) = 0 from the bitmask
          a.e.bits = md.Fbits; a.e.bits_mode = 2; a.e.bits_ld = rows;
        } else {
          a.e.mask = view(md.F, dt, f, 1);
        }
        // db_1 = column sums of dF: 32-row partial sums folded in the dgrad's TMA-store epilogue
        bool db1_fused = false;
        if (c->tune.fuse_db && dt == BF16 && c->csum) a.e.csum = c->csum;
        RET(G_csum(a, c, st, "attn.ffn2_dgrad", &db1_fused));
        RET(ready());   // dF
        {
          Gemm w1 = mk(f, d, (int)rows, 1, operand(dF, dt, 1, f), operand(md.Z1, dt, 1, d), view(gp(md.W1), F32, d, 1));
          w1.e.accumulate = 1;
          RET(G_(w1, c, sd, "attn.ffn1_wgrad", ws2));
          if (db1_fused)
            KTS(sd, "attn.bias_grad", 0, (double)((rows + 31) / 32) * f * 4,
                colsum_add(c->csum, F32, (rows + 31) / 32, f, f, gp(md.b1), red2, c->red_bytes, sd));
          else
            KTS(sd, "attn.bias_grad", 0, (double)rows * f * es, colsum_add(dF, dt, rows, f, f, gp(md.b1), red2, c->red_bytes, sd));
        }
        Gemm z1 = mk((int)rows, d, f, 1, operand(dF, dt, f, 1), operand(p(md.W1), dt, 1, d), view(c->rtmp, F32, d, 1));
        z1.e.resid = view(dR2, dt, d, 1);
        RET(G_(z1, c, st, "attn.ffn1_dgrad"));
        void* dR1 = c->tB;   // dT no longer needed
        KT("attn.ln1_bwd", 0, (double)rows * d * (2 * es + 12), ln_bwd(c->rtmp, F32, md.R1, md.mu1, md.rs1, p(md.g1), dt, rows, d, dR1, dt, acc, 2, gp(md.g1), gp(md.be1),
                  c->red, c->red_bytes, st));
        RET(ready());   // dR1
        {
          Gemm wo = mk(d, d, (int)rows, 1, operand(dR1, dt, 1, d), operand(md.O, dt, 1, d), view(gp(md.Wo), F32, d, 1));
          wo.e.accumulate = 1;
          RET(G_(wo, c, sd, "attn.out_wgrad", ws2));
          KTS(sd, "attn.bias_grad", 0, (double)rows * d * es, colsum_add(dR1, dt, rows, d, d, gp(md.bo), red2, c->red_bytes, sd));
        }
        void* dO = c->tE;
        Gemm go = mk((int)rows, d, d, 1, operand(dR1, dt, d, 1), operand(p(md.Wo), dt, 1, d), view(dO, dt, d, 1));
        RET(G_(go, c, st, "attn.out_dgrad"));
        // attention core backward
        char* dQKV = (char*)c->tF;   // [rows, 3d]
        if (attn::fused_ok(dt, B, H, mi, d)) {
          // B6 core fused: S and P recomputed on chip, dV, dP, dS, dQ, dK per (sample, head)
          ProfScope ps(c, "attn.core_bwd", 10.0 * B * H * (double)mi * mi * dh, (double)B * mi * 7 * d * es, st);
          CK(attn::core_bwd(QKV, dO, dQKV, B, H, mi, d, st));
          if (ps.rec >= 0) c->recs[ps.rec].tc = 1;
        } else {
          const int mp = (mi + 7) / 8 * 8;
          Gemm dv = mk(mi, dh, mi, B * H, operand(md.P, dt, 1, mp, (int64_t)mi * mp),
                       operand(dO, dt, 1, d, (int64_t)mi * d, dh, H),
                       view(dQKV + 2 * (int64_t)d * es, dt, s3, 1, mi * s3, dh, H));
          RET(G_(dv, c, st, "attn.dv"));
          Gemm dp = mk(mi, mi, dh, B * H, operand(dO, dt, d, 1, (int64_t)mi * d, dh, H),
                       operand(QKV + 2 * (int64_t)d * es, dt, s3, 1, mi * s3, dh, H),
                       view(c->big, F32, mp, 1, (int64_t)mi * mp));
          RET(G_(dp, c, st, "attn.dp"));
          KT("attn.softmax_bwd", 0, (double)B * H * mi * mi * (4 + 2 * es), softmax_bwd(md.P, c->big, c->tD, dt, (int64_t)B * H * mi, mi, mp, 1.f / sqrtf((float)dh), st));
          Gemm dq = mk(mi, dh, mi, B * H, operand(c->tD, dt, mp, 1, (int64_t)mi * mp),
                       operand(QKV + (int64_t)d * es, dt, 1, s3, mi * s3, dh, H),
                       view(dQKV, dt, s3, 1, mi * s3, dh, H));
          RET(G_(dq, c, st, "attn.dq"));
          Gemm dk = mk(mi, dh, mi, B * H, operand(c->tD, dt, 1, mp, (int64_t)mi * mp),
                       operand(QKV, dt, 1, s3, mi * s3, dh, H),
                       view(dQKV + (int64_t)d * es, dt, s3, 1, mi * s3, dh, H));
          RET(G_(dk, c, st, "attn.dk"));
        }
        RET(ready());   // dQKV
        {
          Gemm gw = mk(3 * d, d, (int)rows, 1, operand(dQKV, dt, 1, s3), operand(X, dt, 1, d), view(gp(md.Wq), F32, d, 1));
          gw.e.accumulate = 1;
          RET(G_(gw, c, sd, "attn.qkv_wgrad", ws2));
          KTS(sd, "attn.bias_grad", 0, (double)rows * d * es, colsum_add(dQKV, dt, rows, d, s3, gp(md.bq), red2, c->red_bytes, sd));
          KTS(sd, "attn.bias_grad", 0, (double)rows * d * es, colsum_add(dQKV + 2 * (int64_t)d * es, dt, rows, d, s3, gp(md.bv), red2, c->red_bytes, sd));
        }
        Gemm gx = mk((int)rows, d, 3 * d, 1, operand(dQKV, dt, s3, 1), operand(p(md.Wq), dt, 1, d), view(acc, F32, d, 1));
        gx.e.accumulate = 1;
        RET(G_(gx, c, st, "attn.qkv_dgrad"));
        RET(join());
        break;
      }
      case DHEN_DCN_LIT: {   // R31: dW = sum_b G_b dU_b^T, db = sum_b dU_b (side); dG_b = dU_b^T W^T, dX += X (dG + dG^T)
        RET(fork());
        Gemm gw = mk(d, l, B * d, 1, operand(md.G, dt, d, 1, 0, 0, 1, d, (int64_t)d * d),
                     operand(dU, dt, d, 1, 0, 0, 1, d, ldU), view(gp(md.W), F32, l, 1));
        gw.e.accumulate = 1;
        RET(G_(gw, c, sd, "dcnl.wgrad", ws2));
        KTS(sd, "dcnl.bias_grad", 0, (double)B * l * d * es, colsum_add(dU, dt, B, l * d, ldU, gp(md.b), red2, c->red_bytes, sd));
        Gemm gg = mk(d, d, l, B, operand(dU, dt, 1, d, ldU), operand(p(md.W), dt, l, 1), view(md.dGf, F32, d, 1, (int64_t)d * d));
        RET(G_(gg, c, st, "dcnl.dG"));
        KT("dcnl.sym", 0, (double)B * d * d * (4 + es), sym_add(md.dGf, md.S, dt, B, d, st));
        Gemm gx = mk(mi, d, d, B, operand(X, dt, d, 1, (int64_t)mi * d), operand(md.S, dt, 1, d, (int64_t)d * d),
                     view(acc, F32, d, 1, (int64_t)mi * d));
        gx.e.accumulate = 1;
        RET(G_(gx, c, st, "dcnl.dgrad"));
        RET(join());
        break;
      }
      case DHEN_MLP: {   // B9
        const int h1 = md.s.mlp_hidden[0], h2 = md.s.mlp_hidden[1];
        const int K1 = mi * d;
        RET(fork());
        Gemm wm = mk(l * d, h2, B, 1, operand(dU, dt, 1, ldU), operand(md.h2, dt, 1, h2), view(gp(md.Wm), F32, h2, 1));
        wm.e.accumulate = 1;
        RET(G_(wm, c, sd, "mlp.proj_wgrad", ws2));
        void* dh2 = md.dh2;
        Gemm a = mk(B, h2, l * d, 1, operand(dU, dt, ldU, 1), operand(p(md.Wm), dt, 1, h2), view(dh2, dt, h2, 1));
        a.e.mask = view(md.h2, dt, h2, 1);
        RET(G_(a, c, st, "mlp.proj_dgrad"));
        if (sd != st) { CK(cudaEventRecord(c->ev_sx, st)); CK(cudaStreamWaitEvent(sd, c->ev_sx, 0)); }   // dh2 ready
        Gemm w2 = mk(h2, h1, B, 1, operand(dh2, dt, 1, h2), operand(md.h1, dt, 1, h1), view(gp(md.W2), F32, h1, 1));
        w2.e.accumulate = 1;
        RET(G_(w2, c, sd, "mlp.fc2_wgrad", ws2));
        KTS(sd, "mlp.bias_grad", 0, (double)B * h2 * es, colsum_add(dh2, dt, B, h2, h2, gp(md.b2), red2, c->red_bytes, sd));
        void* dh1 = md.dh1;
        Gemm b1 = mk(B, h1, h2, 1, operand(dh2, dt, h2, 1), operand(p(md.W2), dt, 1, h1), view(dh1, dt, h1, 1));
        b1.e.mask = view(md.h1, dt, h1, 1);
        RET(G_(b1, c, st, "mlp.fc2_dgrad"));
        if (sd != st) { CK(cudaEventRecord(c->ev_sx, st)); CK(cudaStreamWaitEvent(sd, c->ev_sx, 0)); }   // dh1 ready
        Gemm w1 = mk(h1, K1, B, 1, operand(dh1, dt, 1, h1), operand(X, dt, 1, K1), view(gp(md.W1), F32, K1, 1));
        w1.e.accumulate = 1;
        RET(G_(w1, c, sd, "mlp.fc1_wgrad", ws2));
        KTS(sd, "mlp.bias_grad", 0, (double)B * h1 * es, colsum_add(dh1, dt, B, h1, h1, gp(md.b1), red2, c->red_bytes, sd));
        Gemm gx = mk(B, K1, h1, 1, operand(dh1, dt, h1, 1), operand(p(md.W1), dt, 1, K1), view(acc, F32, K1, 1));
        gx.e.accumulate = 1;
        if (take_dR) { gx.e.accumulate = 0; gx.e.resid = view(c->dR, dt, K1, 1); }
        if (emit_dX) {   // dX = (dR | acc) + dh1 W1
          if (!take_dR) gx.e.resid = view(acc, F32, K1, 1);
          gx.e.accumulate = 0;
          gx.c = view(dX, dt, K1, 1);
        }
        RET(G_(gx, c, st, "mlp.fc1_dgrad"));
        RET(join());
        break;
      }
    }
  }
  RET(real_join());   // the layer's side-stream work is done before anything after the layer
  if (route) {   // R38: the injected tokens' gradient, then dX = shortcut part + the modules' first m_in tokens (+ dD)
    const int nD = c->cfg.dense_tokens, m_l = Lr.m_in;
    if (Lr.inj) KT("layer.inject_bwd", 0, (double)B * nD * d * 12, inject_dD(acc, B, m_l, nD, d, c->dD, st));
    if (dX)
      KT("layer.dx_cast", 0, (double)B * m_l * d * (8 + es),
         inject_final(acc_sc, acc, mi, n == 0 ? c->dD : nullptr, n == 0 ? nD : 0, B, m_l, d, dX, dt, st));
  } else if (dX && !last_dX) {
    KT("layer.dx_cast", 0, (double)rows * d * (4 + es), cast(acc, F32, dX, dt, rows * d, st));
  }
  RET(release(c, n, st));
  RET(reduce_grads(c, n, st));
  return DHEN_OK;
}

// ------------------------------------------------------------------ block-diagonal token maps, per step
// Single GPU, bf16: the compute weights are fixed for the whole step, so every layer's block-diagonal maps
// (forward packed token projection, DCN backward packed dT) are built up front in ONE launch instead of one
// small launch per module and direction.  The flags are cleared when the step ends (SGD changes W_u).
static dhen_status prebuild_bd(dhen_ctx* c, int B, cudaStream_t st) {
  if (!c->tune.bd_pre || c->dist.world != 1 || c->dt != BF16) return DHEN_OK;
  BdJobs jobs;
  jobs.n = 0;
  for (int n = 0; n < c->cfg.n_layers; ++n) {
    Layer& Lr = c->L[n];
    const int mi = Lr.m_in;
    void* pbase;
    RET(comp_params(c, n, st, &pbase));
    PP p{(char*)pbase, c->es};
    const bool lnf = layer_lnf(c, n, B);
    for (Mod& md : Lr.mods) {
      const int l = md.s.l;
      const int64_t wu = md.s.kind == DHEN_LINEAR ? md.W : md.Wu;
      const bool tm = md.s.kind == DHEN_LINEAR || md.s.kind == DHEN_DCN || md.s.kind == DHEN_DCN_FULL ||
                      md.s.kind == DHEN_CONV || md.s.kind == DHEN_ATTN;
      if (tm && lnf && md.bdT && jobs.n < 32) {
        jobs.job[jobs.n++] = {(const __nv_bfloat16*)p(wu), (__nv_bfloat16*)md.bdT, mi, l, 128 / l, 1};
        md.bdT_pre = true;
      }
      if ((md.s.kind == DHEN_DCN || md.s.kind == DHEN_DCN_FULL) && md.bdg && dcn_pack(c, mi, l, B) && jobs.n < 32) {
        jobs.job[jobs.n++] = {(const __nv_bfloat16*)p(md.Wu), (__nv_bfloat16*)md.bdg, mi, l, 128 / std::max(mi, 1), 0};
        md.bdg_pre = true;
      }
    }
  }
  KT("bdiag.all", 0, 0.0, blockdiag_multi(jobs, st));
  return DHEN_OK;
}
static void clear_bd(dhen_ctx* c) {
  for (Layer& Lr : c->L)
    for (Mod& md : Lr.mods) md.bdT_pre = md.bdg_pre = false;
}

// ------------------------------------------------------------------ head
static dhen_status head(dhen_ctx* c, const void* YN, int mN, const float* labels, int B, int Bg, void* dY, float* loss,
                        int do_bwd, bool keep_w, cudaStream_t st) {
  const int gi = c->cfg.n_layers;
  void* pbase;
  RET(comp_params(c, gi, st, &pbase));
  PP p{(char*)pbase, c->es};
  Group& G = c->G[gi];
  // the head's parameter / loss sums trail on the side stream (the first backward layer's module joins bring
  // it back before anything reads them; with collectives the reduce-scatter also waits for it)
  cudaStream_t sr = (c->tune.overlap && c->tune.trail && !serial_prof(c)) ? c->side_st : st;
  KT("head", 0, (double)B * mN * c->d * c->es * (do_bwd ? 2 : 1), head_fwd_bwd(YN, p(0), p(G.toff[1]), c->dt, labels, B, mN, c->d, Bg, dY, c->dt, c->pooled, c->z, c->lossb, c->dz, loss,
                  G.grad, G.grad + G.toff[1], do_bwd, st, sr, c->ev_red));
  // FSDP: the gathered slot is reused by the next all-gather; the last layer's LN backward reads w_h from a copy
  if (keep_w && sharded(c)) CK(cudaMemcpyAsync(c->headw, p(0), (size_t)c->d * c->es, cudaMemcpyDeviceToDevice, st));
  RET(release(c, gi, st));
  if (do_bwd) RET(reduce_grads(c, gi, st, sr));
  return DHEN_OK;
}

// ------------------------------------------------------------------ C ABI
static bool aligned16(const void* p) { return p && (((uintptr_t)p) & 15) == 0; }
static cudaStream_t S(void* s) { return (cudaStream_t)s; }

extern "C" {

const char* dhen_last_error(void) { return t_err.c_str(); }

dhen_status dhen_validate(const dhen_config* cfg) { return validate(cfg); }

static dhen_status make_ctx(const dhen_config* cfg, const dhen_dist* dist, dhen_ctx* c) {
  RET(validate(cfg));
  dhen_dist dd;
  if (dist) dd = *dist; else { memset(&dd, 0, sizeof dd); dd.world = 1; dd.fsdp = 1; }
  if (dd.world < 1 || dd.rank < 0 || dd.rank >= dd.world)
    return fail(DHEN_E_CONFIG, "dhen: rank=%d world=%d", dd.rank, dd.world);
  if (dd.backend != 0 && dd.backend != 1) return fail(DHEN_E_CONFIG, "dhen: collective backend=%d (0 NCCL, 1 loopback)", dd.backend);
  c->cfg = *cfg;
  if (c->cfg.ln_eps <= 0.f) c->cfg.ln_eps = 1e-5f;
  if (c->cfg.adam_beta1 <= 0.f) c->cfg.adam_beta1 = 0.9f;
  if (c->cfg.adam_beta2 <= 0.f) c->cfg.adam_beta2 = 0.999f;
  if (c->cfg.adam_eps <= 0.f) c->cfg.adam_eps = 1e-8f;
  c->mods_cfg.resize(cfg->n_layers);
  c->layers_cfg.resize(cfg->n_layers);
  for (int n = 0; n < cfg->n_layers; ++n) {
    c->mods_cfg[n].assign(cfg->layers[n].modules, cfg->layers[n].modules + cfg->layers[n].n_modules);
    c->layers_cfg[n].n_modules = cfg->layers[n].n_modules;
    c->layers_cfg[n].ensemble = cfg->layers[n].ensemble;
    c->layers_cfg[n].dense_in = cfg->layers[n].dense_in;
    c->layers_cfg[n].modules = c->mods_cfg[n].data();
  }
  c->cfg.layers = c->layers_cfg.data();
  c->dist = dd;
  c->dt = cfg->dtype == DHEN_BF16 ? BF16 : F32;
  c->es = c->dt == BF16 ? 2 : 4;
  c->d = cfg->d;
  c->Bmax = cfg->batch_max_local;
  return DHEN_OK;
}

dhen_status dhen_sizes(const dhen_config* cfg, const dhen_dist* dist, size_t* state_bytes, size_t* work_bytes) {
  dhen_ctx c;
  RET(make_ctx(cfg, dist, &c));
  Carver s(nullptr), w(nullptr);
  plan(&c, s, w);
  if (state_bytes) *state_bytes = s.off + 256;
  if (work_bytes) *work_bytes = w.off + 256;
  return DHEN_OK;
}

dhen_status dhen_group_numel(const dhen_config* cfg, const dhen_dist* dist, int group, size_t* numel, size_t* shard) {
  dhen_ctx c;
  RET(make_ctx(cfg, dist, &c));
  Carver s(nullptr), w(nullptr);
  plan(&c, s, w);
  if (group < 0 || group > cfg->n_layers) return fail(DHEN_E_SHAPE, "dhen_group_numel: group=%d of %d", group, cfg->n_layers + 1);
  if (numel) *numel = (size_t)c.G[group].ncanon;
  if (shard) *shard = (size_t)c.G[group].shard;
  return DHEN_OK;
}

dhen_status dhen_loopback_id(unsigned char out[128]) {
  if (!out) return fail(DHEN_E_ALIGN, "dhen_loopback_id: out is NULL");
  loopback_new_id(out);
  return DHEN_OK;
}

unsigned long long dhen_comm_bytes(const dhen_ctx* c) { return c && c->comm ? c->comm->bytes : 0ull; }

dhen_status dhen_nccl_id(unsigned char out[128]) {
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  memcpy(out, id.internal, 128);
  return DHEN_OK;
}

dhen_status dhen_init(const dhen_config* cfg, const dhen_dist* dist, void* state, size_t state_bytes, void* work,
                      size_t work_bytes, void* stream, dhen_ctx** out) {
  if (!out) return fail(DHEN_E_ALIGN, "dhen_init: out is NULL");
  *out = nullptr;
  dhen_ctx* c = new dhen_ctx();
  dhen_status s0 = make_ctx(cfg, dist, c);
  if (s0 != DHEN_OK) { delete c; return s0; }
  if (!aligned16(state) || !aligned16(work)) { delete c; return fail(DHEN_E_ALIGN, "dhen_init: state=%p work=%p not 16-B aligned", state, work); }
  Carver sz(nullptr), wz(nullptr);
  plan(c, sz, wz);
  if (state_bytes < sz.off || work_bytes < wz.off) {
    size_t a = sz.off, b = wz.off;
    delete c;
    return fail(DHEN_E_NOMEM, "dhen_init: state %zu < %zu or work %zu < %zu bytes", state_bytes, a, work_bytes, b);
  }
  // align bases to 256
  Carver s((void*)(((uintptr_t)state + 255) & ~uintptr_t(255))), w((void*)(((uintptr_t)work + 255) & ~uintptr_t(255)));
  if (((uintptr_t)state & 255) || ((uintptr_t)work & 255)) {
    if (state_bytes < sz.off + 256 || work_bytes < wz.off + 256) { delete c; return fail(DHEN_E_NOMEM, "dhen_init: buffers too small after alignment"); }
  }
  plan(c, s, w);
  {
    bool ok = cudaStreamCreateWithFlags(&c->side_st, cudaStreamNonBlocking) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_sf, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_sx, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_sj, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_red, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) { dhen_destroy(c); return fail(DHEN_E_CUDA, "dhen_init: side stream creation failed"); }
  }
  if (c->dist.world > 1) {
    std::string why;
    c->comm = comm_create(c->dist.backend, c->dist.nccl_id, c->dist.world, c->dist.rank, &why);
    if (!c->comm) { dhen_destroy(c); return fail(DHEN_E_NCCL, "dhen_init: collective backend %d: %s", c->dist.backend, why.c_str()); }
    bool ok = cudaStreamCreateWithFlags(&c->comm_st, cudaStreamNonBlocking) == cudaSuccess;
    for (int k = 0; k < 2; ++k) {
      ok = ok && cudaEventCreateWithFlags(&c->ev_ag[k], cudaEventDisableTiming) == cudaSuccess;
      ok = ok && cudaEventCreateWithFlags(&c->ev_use[k], cudaEventDisableTiming) == cudaSuccess;
    }
    ok = ok && cudaEventCreateWithFlags(&c->ev_grad, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_grad2, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_cfork, cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; k < 2; ++k) ok = ok && cudaEventCreateWithFlags(&c->ev_rs[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) { dhen_destroy(c); return fail(DHEN_E_CUDA, "dhen_init: stream/event creation failed"); }
  }
  // parameter init: every rank initialises its own slice of the canonical vector
  const unsigned long long launches_before = g_launches;
  cudaStream_t st = S(stream);
  for (size_t gi = 0; gi < c->G.size(); ++gi) {
    Group& g = c->G[gi];
    const int64_t lo = (c->dist.world > 1 && c->dist.fsdp) ? (int64_t)c->dist.rank * g.shard : 0;
    const int64_t hi = lo + g.shard;
    cudaError_t e = cudaMemsetAsync(g.master, 0, g.shard * 4, st);
    if (e != cudaSuccess) { delete c; return fail(DHEN_E_CUDA, "dhen_init: %s", cudaGetErrorString(e)); }
    for (size_t t = 0; t < g.toff.size(); ++t) {
      int64_t a = std::max(lo, g.toff[t]), b = std::min(hi, g.toff[t] + g.tn[t]);
      if (a >= b) continue;
      // uniform values depend on the tensor's global index only (same params at any world size)
      if (g.tinit[t] == 0) {
        cudaError_t e2 = init_uniform(g.master + (a - lo), b - a, g.tbound[t], c->cfg.seed, gi * 4096 + t, a - g.toff[t], st);
        if (e2 != cudaSuccess) { delete c; return fail(DHEN_E_CUDA, "dhen_init: %s", cudaGetErrorString(e2)); }
      } else {
        cudaError_t e2 = fill(g.master + (a - lo), b - a, g.tinit[t] == 1 ? 1.f : 0.f, st);
        if (e2 != cudaSuccess) { delete c; return fail(DHEN_E_CUDA, "dhen_init: %s", cudaGetErrorString(e2)); }
      }
    }
    cudaError_t e3 = sgd_cast(g.master, nullptr, 0.f, g.comp, c->dt, g.shard, st);
    if (e3 != cudaSuccess) { delete c; return fail(DHEN_E_CUDA, "dhen_init: %s", cudaGetErrorString(e3)); }
    e3 = cudaMemsetAsync(g.grad, 0, g.npad * 4, st);
    if (e3 == cudaSuccess && g.adam_m) e3 = cudaMemsetAsync(g.adam_m, 0, g.shard * (c->cfg.optimizer == 2 ? 2 : 4), st);
    if (e3 == cudaSuccess && g.adam_v) e3 = cudaMemsetAsync(g.adam_v, 0, g.shard * (c->cfg.optimizer == 2 ? 2 : 4), st);
    if (e3 != cudaSuccess) { delete c; return fail(DHEN_E_CUDA, "dhen_init: %s", cudaGetErrorString(e3)); }
  }
  if (c->adam_t && cudaMemsetAsync(c->adam_t, 0, sizeof(int), st) != cudaSuccess) {
    delete c;
    return fail(DHEN_E_CUDA, "dhen_init: adam step counter");
  }
  c->launches0 = launches_before;
  if (fence_params(c, st) != DHEN_OK) { dhen_destroy(c); return DHEN_E_CUDA; }
  *out = c;
  return DHEN_OK;
}

void dhen_destroy(dhen_ctx* c) {
  if (!c) return;
  for (auto e : c->events) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    if (c->ev_ag[k]) cudaEventDestroy(c->ev_ag[k]);
    if (c->ev_use[k]) cudaEventDestroy(c->ev_use[k]);
  }
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->cap_st) cudaStreamDestroy(c->cap_st);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_sf) cudaEventDestroy(c->ev_sf);
  if (c->ev_sx) cudaEventDestroy(c->ev_sx);
  if (c->ev_sj) cudaEventDestroy(c->ev_sj);
  if (c->ev_red) cudaEventDestroy(c->ev_red);
  if (c->side_st) cudaStreamDestroy(c->side_st);
  if (c->ev_grad) cudaEventDestroy(c->ev_grad);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (c->ev_grad2) cudaEventDestroy(c->ev_grad2);
  if (c->ev_cfork) cudaEventDestroy(c->ev_cfork);
  for (int k = 0; k < 2; ++k) if (c->ev_rs[k]) cudaEventDestroy(c->ev_rs[k]);
  if (c->comm_st) cudaStreamDestroy(c->comm_st);
  for (int k = 0; k < 2; ++k) {
    if (c->hx[k]) cudaFree(c->hx[k]);
    if (c->hy[k]) cudaFree(c->hy[k]);
    if (c->hev_up[k]) cudaEventDestroy(c->hev_up[k]);
    if (c->hev_free[k]) cudaEventDestroy(c->hev_free[k]);
  }
  if (c->hxin) cudaFree(c->hxin);
  if (c->hyin) cudaFree(c->hyin);
  if (c->hloss) cudaFree(c->hloss);
  if (c->hcp) cudaStreamDestroy(c->hcp);
  delete c->comm;
  delete c;
}

unsigned long long dhen_launch_count(const dhen_ctx* c) { return c ? g_launches - c->launches0 : 0; }

dhen_status dhen_debug_gemm(const long long* q, const void* A, const void* Bp, void* Cp, int ab_dt, int c_dt, int path,
                            void* ws, size_t ws_bytes, void* stream) {
  if (!q || !A || !Bp || !Cp) return fail(DHEN_E_ALIGN, "dhen_debug_gemm: NULL argument");
  const int abt = ab_dt == DHEN_BF16 ? BF16 : F32, ct = c_dt == DHEN_BF16 ? BF16 : F32;
  Gemm g = mk((int)q[0], (int)q[1], (int)q[2], (int)q[3],
              operand(A, abt, q[4], q[5], q[6], q[7], (int)q[8], (int)q[9], q[10]),
              operand(Bp, abt, q[11], q[12], q[13], q[14], (int)q[15], (int)q[16], q[17]),
              view(Cp, ct, q[18], q[19], q[20], q[21], (int)q[22]));
  g.e.accumulate = (int)q[23];
  g.a.mdiv = (int)q[24]; g.a.s_mo = q[25];
  g.b.mdiv = (int)q[26]; g.b.s_mo = q[27];
  g.c.rdiv = (int)q[28]; g.c.rs_o = q[29];
  Workspace w;
  w.ptr = (float*)ws;
  w.bytes = ws_bytes;
  dhen::g_gemm_force = path >= 3 ? 2 : path;
  const int pair_prev = dhen::g_gemm_pair;
  dhen::g_gemm_pair = path == 3 ? 1 : path == 4 ? 0 : pair_prev;
  cudaError_t e = gemm_run(g, w, S(stream));
  const int used_tc = g_last_gemm_tc;
  dhen::g_gemm_force = -1;
  dhen::g_gemm_pair = pair_prev;
  if (e == cudaErrorNotSupported) return fail(DHEN_E_CONFIG, "dhen_debug_gemm: layout not supported on this path");
  CK(e);
  return used_tc ? DHEN_OK : DHEN_OK;
}

int dhen_debug_last_gemm_tc(void) { return g_last_gemm_tc; }

dhen_status dhen_debug_gemm_epi(const long long* q, const void* A, const void* Bp, void* Cp, int ab_dt, int c_dt,
                                int path, void* ws, size_t ws_bytes, int mode, const void* E, const void* bias,
                                void* aux, void* stream) {
  if (!q || !A || !Bp || !Cp) return fail(DHEN_E_ALIGN, "dhen_debug_gemm_epi: NULL argument");
  const int abt = ab_dt == DHEN_BF16 ? BF16 : F32, ct = c_dt == DHEN_BF16 ? BF16 : F32;
  Gemm g = mk((int)q[0], (int)q[1], (int)q[2], (int)q[3],
              operand(A, abt, q[4], q[5], q[6], q[7], (int)q[8], (int)q[9], q[10]),
              operand(Bp, abt, q[11], q[12], q[13], q[14], (int)q[15], (int)q[16], q[17]),
              view(Cp, ct, q[18], q[19], q[20], q[21], (int)q[22]));
  g.e.accumulate = (int)q[23];
  g.a.mdiv = (int)q[24]; g.a.s_mo = q[25];
  g.b.mdiv = (int)q[26]; g.b.s_mo = q[27];
  g.c.rdiv = (int)q[28]; g.c.rs_o = q[29];
  View ev = g.c;   // the extra operand shares C's geometry, in bf16
  ev.dt = BF16;
  ev.ptr = const_cast<void*>(E);
  if (bias) { g.e.bias = bias; g.e.bias_dt = BF16; }
  switch (mode) {   // 1 mask, 2 residual, 3 DCN cross (+ aux), 4 relu, 5 relu + bitmask out (aux), 6 bitmask in (aux)
    case 1: g.e.mask = ev; break;
    case 2: g.e.resid = ev; break;
    case 3: g.e.cross = ev; if (aux) { g.e.aux = ev; g.e.aux.ptr = aux; } break;
    case 4: g.e.relu = 1; break;
    case 5: g.e.relu = 1; g.e.bits = (uint32_t*)aux; g.e.bits_mode = 1; g.e.bits_ld = g.M; break;
    case 6: g.e.bits = (uint32_t*)aux; g.e.bits_mode = 2; g.e.bits_ld = g.M; break;
    default: break;
  }
  Workspace w;
  w.ptr = (float*)ws;
  w.bytes = ws_bytes;
  dhen::g_gemm_force = path >= 3 ? 2 : path;
  const int pair_prev = dhen::g_gemm_pair;
  dhen::g_gemm_pair = path == 3 ? 1 : path == 4 ? 0 : pair_prev;
  cudaError_t e = gemm_run(g, w, S(stream));
  dhen::g_gemm_force = -1;
  dhen::g_gemm_pair = pair_prev;
  if (e == cudaErrorNotSupported) return fail(DHEN_E_CONFIG, "dhen_debug_gemm_epi: layout not supported on this path");
  CK(e);
  return DHEN_OK;
}

void dhen_debug_gemm_trace(void* dev_buf) { g_gemm_trace = (long long*)dev_buf; }

dhen_status dhen_debug_profile_trace(dhen_ctx* c, const char* path) {
  if (!c || !path) return fail(DHEN_E_STATE, "dhen_debug_profile_trace: ctx or path is NULL");
  FILE* fp = fopen(path, "w");
  if (!fp) return fail(DHEN_E_CONFIG, "dhen_debug_profile_trace: cannot open %s", path);
  std::vector<cudaStream_t> sts;
  for (auto& r : c->recs) {
    CK(cudaEventSynchronize(c->events[r.e1]));
    float t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&t0, c->events[c->recs[0].e0], c->events[r.e0]);
    cudaEventElapsedTime(&t1, c->events[c->recs[0].e0], c->events[r.e1]);
    size_t si = 0;
    for (; si < sts.size(); ++si) if (sts[si] == r.st) break;
    if (si == sts.size()) sts.push_back(r.st);
    fprintf(fp, "%s,%zu,%.4f,%.4f\n", r.tag, si, t0, t1);
  }
  fclose(fp);
  return DHEN_OK;
}

void dhen_tuning_default(dhen_tuning* t) { if (t) *t = tuning_default(); }

dhen_status dhen_set_tuning(dhen_ctx* c, const dhen_tuning* t) {
  if (!c || !t) return fail(DHEN_E_STATE, "dhen_set_tuning: ctx or tuning is NULL");
  const int bits[] = {t->overlap, t->defer_join, t->ln_fuse, t->first_writer, t->relu_bits, t->fuse_db, t->vdy,
                      t->trail, t->bd_pre, t->tstore, t->attn_fused, t->pdl, t->gemm_simt, t->dcn_fused, t->dcn_tma, t->ln_tma, t->resid_tma};
  for (int b : bits)
    if (b != 0 && b != 1) return fail(DHEN_E_CONFIG, "dhen_set_tuning: a 0/1 switch is %d", b);
  if (t->bn_max != 64 && t->bn_max != 128 && t->bn_max != 256)
    return fail(DHEN_E_CONFIG, "dhen_set_tuning: bn_max=%d (64, 128 or 256)", t->bn_max);
  if (t->wres < 0 || t->wres > 2) return fail(DHEN_E_CONFIG, "dhen_set_tuning: wres=%d (0, 1 or 2)", t->wres);
  if (t->l2_prefetch < 0 || t->l2_prefetch > 4)
    return fail(DHEN_E_CONFIG, "dhen_set_tuning: l2_prefetch=%d (0..4)", t->l2_prefetch);
  if (t->sym < -1 || t->sym > 2 || t->pair < -1 || t->pair > 1 || t->pair_k < 0)
    return fail(DHEN_E_CONFIG, "dhen_set_tuning: sym=%d pair=%d pair_k=%d", t->sym, t->pair, t->pair_k);
  c->tune = *t;
  if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }   // the captured step baked the old switches in
  c->graph_off = false;
  return DHEN_OK;
}

dhen_status dhen_get_tuning(const dhen_ctx* c, dhen_tuning* t) {
  if (!c || !t) return fail(DHEN_E_STATE, "dhen_get_tuning: ctx or tuning is NULL");
  *t = c->tune;
  return DHEN_OK;
}

dhen_status dhen_profile(dhen_ctx* c, int enable) {
  if (!c) return fail(DHEN_E_STATE, "dhen_profile: ctx is NULL");
  c->prof = enable != 0;
  c->prof_mode = enable == 2 ? 2 : 1;
  if (enable) { c->recs.clear(); c->next_event = 0; }
  return DHEN_OK;
}

dhen_status dhen_profile_read(dhen_ctx* c, dhen_op_stat* out, int cap, int* n) {
  if (!c || !n) return fail(DHEN_E_STATE, "dhen_profile_read: ctx or n is NULL");
  std::vector<dhen_op_stat> agg;
  for (auto& r : c->recs) {
    CK(cudaEventSynchronize(c->events[r.e1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->events[r.e0], c->events[r.e1]));
    size_t k = 0;
    for (; k < agg.size(); ++k) if (!strncmp(agg[k].name, r.tag, sizeof agg[k].name)) break;
    if (k == agg.size()) {
      dhen_op_stat z;
      memset(&z, 0, sizeof z);
      strncpy(z.name, r.tag, sizeof z.name - 1);
      agg.push_back(z);
    }
    agg[k].launches += 1;
    agg[k].ms += ms;
    agg[k].flops += r.flops;
    agg[k].bytes += r.bytes;
    agg[k].tc_launches += r.tc ? 1 : 0;
  }
  *n = (int)agg.size();
  for (int k = 0; k < (int)agg.size() && k < cap; ++k) out[k] = agg[k];
  return DHEN_OK;
}

dhen_status dhen_zero_grad(dhen_ctx* c, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_zero_grad: ctx is NULL");
  for (auto& g : c->G) {
    CK(cudaMemsetAsync(g.grad, 0, g.npad * 4, S(stream)));
    if (g.gshard) CK(cudaMemsetAsync(g.gshard, 0, g.shard * 4, S(stream)));
  }
  return DHEN_OK;
}

dhen_status dhen_layer_fwd(dhen_ctx* c, int n, const void* x, void* y, int B, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_layer_fwd: ctx is NULL");
  TuneScope ts_(&c->tune);
  if (n < 0 || n >= c->cfg.n_layers) return fail(DHEN_E_SHAPE, "dhen_layer_fwd: layer=%d of %d", n, c->cfg.n_layers);
  if (B < 1 || B > c->Bmax) return fail(DHEN_E_SHAPE, "dhen_layer_fwd: B=%d not in [1, %d]", B, c->Bmax);
  if (!aligned16(x) || !aligned16(y)) return fail(DHEN_E_ALIGN, "dhen_layer_fwd: x=%p y=%p", x, y);
  invalidate_gathered(c);
  clear_bd(c);
  RET(layer_fwd(c, n, x, y, B, S(stream)));
  CK(cudaGetLastError());
  return DHEN_OK;
}

dhen_status dhen_layer_bwd(dhen_ctx* c, int n, const void* dy, void* dx, int B, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_layer_bwd: ctx is NULL");
  TuneScope ts_(&c->tune);
  if (n < 0 || n >= c->cfg.n_layers) return fail(DHEN_E_SHAPE, "dhen_layer_bwd: layer=%d of %d", n, c->cfg.n_layers);
  if (c->L[n].B != B) return fail(DHEN_E_STATE, "dhen_layer_bwd: layer %d has no saved forward at B=%d (saved B=%d)", n, B, c->L[n].B);
  if (!aligned16(dy) || (dx && !aligned16(dx))) return fail(DHEN_E_ALIGN, "dhen_layer_bwd: dy=%p dx=%p", dy, dx);
  invalidate_gathered(c);
  clear_bd(c);
  RET(layer_bwd(c, n, dy, dx, B, S(stream)));
  RET(join_comm(c, S(stream)));
  CK(cudaGetLastError());
  return DHEN_OK;
}

dhen_status dhen_forward(dhen_ctx* c, const void* x0, int B, float* logits, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_forward: ctx is NULL");
  TuneScope ts_(&c->tune);
  if (B < 1 || B > c->Bmax) return fail(DHEN_E_SHAPE, "dhen_forward: B=%d not in [1, %d]", B, c->Bmax);
  if (!aligned16(x0) || !aligned16(logits)) return fail(DHEN_E_ALIGN, "dhen_forward: x0=%p logits=%p", x0, logits);
  cudaStream_t st = S(stream);
  invalidate_gathered(c);
  const void* X = x0;
  for (int n = 0; n < c->cfg.n_layers; ++n) {
    RET(prefetch(c, n));
    RET(prefetch(c, n + 1));          // overlap the next group's all-gather with this layer
    RET(layer_fwd(c, n, X, c->L[n].Y, B, st));
    X = c->L[n].Y;
  }
  RET(head(c, X, c->L.back().m_out, nullptr, B, B, nullptr, nullptr, 0, false, st));
  CK(cudaMemcpyAsync(logits, c->z, (size_t)B * 4, cudaMemcpyDeviceToDevice, st));
  CK(cudaGetLastError());
  return DHEN_OK;
}

dhen_status dhen_train_step(dhen_ctx* c, const void* x0, const float* labels, int B, int Bg, float lr, float* loss,
                            void* dx0, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_train_step: ctx is NULL");
  TuneScope ts_(&c->tune);
  if (B < 1 || B > c->Bmax) return fail(DHEN_E_SHAPE, "dhen_train_step: B=%d not in [1, %d]", B, c->Bmax);
  if (Bg < B) return fail(DHEN_E_SHAPE, "dhen_train_step: B_global=%d < B=%d", Bg, B);
  if (!aligned16(x0) || !aligned16(labels) || (dx0 && !aligned16(dx0)) || (loss && ((uintptr_t)loss & 3)))
    return fail(DHEN_E_ALIGN, "dhen_train_step: x0=%p labels=%p dx0=%p loss=%p", x0, (const void*)labels, dx0, (void*)loss);
  if (!std::isfinite(lr)) return fail(DHEN_E_CONFIG, "dhen_train_step: lr=%g", (double)lr);
  cudaStream_t st = S(stream);
  RET(dhen_zero_grad(c, stream));
  invalidate_gathered(c);
  if (c->dist.world > 1) {
    // the communication stream (and the slot-release events it waits on) start from this step's stream: the
    // collectives are ordered after everything before the step, and a CUDA-graph capture of the step takes
    // the communication stream in with it
    CK(cudaEventRecord(c->ev_cfork, st));
    CK(cudaStreamWaitEvent(c->comm_st, c->ev_cfork, 0));
    for (int k = 0; k < 2; ++k) CK(cudaEventRecord(c->ev_use[k], st));
  }
  const void* X = x0;
  clear_bd(c);
  RET(prebuild_bd(c, B, st));
  for (int n = 0; n < c->cfg.n_layers; ++n) {
    RET(prefetch(c, n));
    RET(prefetch(c, n + 1));          // overlap the next group's all-gather with this layer (F0)
    RET(layer_fwd(c, n, X, c->L[n].Y, B, st));
    X = c->L[n].Y;
  }
  // bf16: the head writes only dz; the last layer's LN backward forms dY = dz w / m itself
  const bool vdy = c->tune.vdy && c->dt == BF16 && c->d % 8 == 0 && c->d >= 32 && c->d <= 256 && (c->d & (c->d - 1)) == 0;
  RET(head(c, X, c->L.back().m_out, labels, B, Bg, vdy ? nullptr : c->dY[0], loss, 1, vdy, st));
  c->vdy_now = vdy;
  int cur = 0;
  for (int n = c->cfg.n_layers - 1; n >= 0; --n) {
    void* dx = n > 0 ? c->dY[cur ^ 1] : dx0;
    RET(prefetch(c, n));
    RET(prefetch(c, n - 1));          // re-gather for backward ahead of use; RS of n runs behind (B11)
    RET(layer_bwd(c, n, c->dY[cur], dx, B, st));
    cur ^= 1;
  }
  RET(join_comm(c, st));
  // B12: the optimizer on the (local shard of the) fp32 masters, refresh the compute copy
  if (c->cfg.optimizer >= 1) {   // Adam (NEXT#3): per group, then the device step counter
    const int mdt = c->cfg.optimizer == 2 ? BF16 : F32;
    for (auto& g : c->G) {
      const float* gr = c->dist.world > 1 ? g.gshard : g.grad;
      KT("adam", 0, (double)g.shard * (12 + 4 * (mdt == BF16 ? 2 : 4) + c->es),
         adam_step(g.master, gr, g.adam_m, g.adam_v, mdt, g.comp, c->dt, g.shard, lr, c->cfg.adam_beta1,
                   c->cfg.adam_beta2, c->cfg.adam_eps, c->adam_t, st));
    }
    CK(adam_count(c->adam_t, st));
    RET(fence_params(c, st));
    clear_bd(c);
    CK(cudaGetLastError());
    return DHEN_OK;
  }
  bool multi = c->dt == BF16 && c->G.size() <= 32;
  for (auto& g : c->G) multi = multi && g.shard % 4 == 0;
  if (multi) {   // every group in one launch
    SgdSegs segs;
    segs.n = 0;
    double bytes = 0;
    for (auto& g : c->G) {
      segs.master[segs.n] = g.master;
      segs.grad[segs.n] = c->dist.world > 1 ? g.gshard : g.grad;
      segs.copy[segs.n] = g.comp;
      segs.n4[segs.n] = g.shard / 4;
      ++segs.n;
      bytes += (double)g.shard * (12 + c->es);
    }
    KT("sgd", 0, bytes, sgd_multi(segs, lr, st));
  } else {
    for (auto& g : c->G) {
      const float* gr = c->dist.world > 1 ? g.gshard : g.grad;
      KT("sgd", 0, (double)g.shard * (12 + c->es), sgd_cast(g.master, gr, lr, g.comp, c->dt, g.shard, st));
    }
  }
  RET(fence_params(c, st));
  clear_bd(c);
  CK(cudaGetLastError());
  return DHEN_OK;
}

// The library keeps every tensor 128-B aligned inside its group (internal layout); the
// caller sees the dense canonical order.  These copy between the two through a host buffer.
static void to_internal(const Group& g, const float* canon, std::vector<float>& pad) {
  pad.assign((size_t)g.npad, 0.f);
  for (size_t t = 0; t < g.toff.size(); ++t)
    memcpy(pad.data() + g.toff[t], canon + g.tcanon[t], (size_t)g.tn[t] * 4);
}
static void to_canonical(const Group& g, const float* pad, float* canon) {
  for (size_t t = 0; t < g.toff.size(); ++t)
    memcpy(canon + g.tcanon[t], pad + g.toff[t], (size_t)g.tn[t] * 4);
}
// full (all ranks) internal vector of a sharded fp32 buffer -> host
static dhen_status gather_f32(dhen_ctx* c, Group& g, const float* shard_or_full, std::vector<float>& pad,
                              cudaStream_t st) {
  pad.assign((size_t)g.npad, 0.f);
  if (c->dist.world > 1 && c->dist.fsdp) {
    if (c->comm->all_gather(shard_or_full, c->gtmp, (size_t)g.shard, F32, st))
      return fail(DHEN_E_NCCL, "all-gather (fp32 host read) (%s): %s", c->comm->name(), c->comm->err.c_str());
    CK(cudaMemcpyAsync(pad.data(), c->gtmp, (size_t)g.npad * 4, cudaMemcpyDeviceToHost, st));
  } else {
    CK(cudaMemcpyAsync(pad.data(), shard_or_full, (size_t)g.n * 4, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return DHEN_OK;
}

dhen_status dhen_train_step_host(dhen_ctx* c, const void* x0_host, const float* labels_host, int B, int Bg, float lr,
                                 float* loss_host, int sync, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_train_step_host: ctx is NULL");
  if (!x0_host || !labels_host || !loss_host)
    return fail(DHEN_E_ALIGN, "dhen_train_step_host: x0_host=%p labels_host=%p loss_host=%p", x0_host,
                (const void*)labels_host, (void*)loss_host);
  if (B < 1 || B > c->Bmax) return fail(DHEN_E_SHAPE, "dhen_train_step_host: B=%d not in [1, %d]", B, c->Bmax);
  cudaStream_t st = S(stream);
  const size_t xrow = (size_t)c->cfg.m0 * c->d * (c->dt == BF16 ? 2 : 4);
  if (!c->hxin) {   // first call: staging slots, input buffers, copy stream, slot events (slots start free)
    for (int k = 0; k < 2; ++k) {
      CK(cudaMalloc(&c->hx[k], xrow * c->Bmax));
      CK(cudaMalloc((void**)&c->hy[k], sizeof(float) * c->Bmax));
      CK(cudaEventCreateWithFlags(&c->hev_up[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->hev_free[k], cudaEventDisableTiming));
      CK(cudaEventRecord(c->hev_free[k], st));
    }
    CK(cudaMalloc(&c->hxin, xrow * c->Bmax));
    CK(cudaMalloc((void**)&c->hyin, sizeof(float) * c->Bmax));
    CK(cudaMalloc((void**)&c->hloss, sizeof(float)));
    CK(cudaStreamCreateWithFlags(&c->hcp, cudaStreamNonBlocking));
  }
  const int s = (int)(c->hcalls & 1);
  // upload into slot s once the step that last moved it out is done with it
  CK(cudaStreamWaitEvent(c->hcp, c->hev_free[s], 0));
  CK(cudaMemcpyAsync(c->hx[s], x0_host, xrow * B, cudaMemcpyHostToDevice, c->hcp));
  CK(cudaMemcpyAsync(c->hy[s], labels_host, sizeof(float) * B, cudaMemcpyHostToDevice, c->hcp));
  CK(cudaEventRecord(c->hev_up[s], c->hcp));
  // into the step's (fixed) input buffers, so the captured step graph is replayed, not re-captured
  CK(cudaStreamWaitEvent(st, c->hev_up[s], 0));
  CK(cudaMemcpyAsync(c->hxin, c->hx[s], xrow * B, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(c->hyin, c->hy[s], sizeof(float) * B, cudaMemcpyDeviceToDevice, st));
  CK(cudaEventRecord(c->hev_free[s], st));
  ++c->hcalls;
  RET(dhen_train_step_graphed(c, c->hxin, c->hyin, B, Bg, lr, c->hloss, nullptr, stream));
  CK(cudaMemcpyAsync(loss_host, c->hloss, sizeof(float), cudaMemcpyDeviceToHost, st));
  if (sync) CK(cudaStreamSynchronize(st));
  return DHEN_OK;
}

dhen_status dhen_train_step_graphed(dhen_ctx* c, const void* x0, const float* labels, int B, int Bg, float lr,
                                    float* loss, void* dx0, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_train_step_graphed: ctx is NULL");
  TuneScope ts_(&c->tune);
  // loopback collectives are host rendezvous between threads (not capturable); a profiled step records events
  if (c->prof || (c->dist.world > 1 && (c->dist.backend != 0 || c->graph_off)))
    return dhen_train_step(c, x0, labels, B, Bg, lr, loss, dx0, stream);
  cudaStream_t st = S(stream);
  const bool same = c->gexec && c->gkey[0] == x0 && c->gkey[1] == labels && c->gkey[2] == loss &&
                    c->gkey[3] == dx0 && c->gkey_B == B && c->gkey_Bg == Bg && c->gkey_lr == lr;
  if (!same) {
    if (c->gexec) { CK(cudaGraphExecDestroy(c->gexec)); c->gexec = nullptr; }
    if (!c->cap_st) {
      CK(cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    // validate + warm (attribute setup, TMA-descriptor paths) eagerly once, then capture
    RET(dhen_train_step(c, x0, labels, B, Bg, lr, loss, dx0, stream));
    CK(cudaStreamSynchronize(st));
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(c->cap_st, cudaStreamCaptureModeThreadLocal));
    const unsigned long long l0 = g_launches;
    dhen_status s0 = dhen_train_step(c, x0, labels, B, Bg, lr, loss, dx0, c->cap_st);
    c->graph_launches = g_launches - l0;
    cudaError_t e = cudaStreamEndCapture(c->cap_st, &graph);
    if (s0 != DHEN_OK || e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      if (c->dist.world > 1) {   // NCCL step not capturable here: every later step runs eagerly (same result)
        (void)cudaGetLastError();
        c->graph_off = true;
        return DHEN_OK;          // this call's step already ran eagerly
      }
      if (s0 != DHEN_OK) return s0;
      CK(e);
    }
    e = cudaGraphInstantiate(&c->gexec, graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    c->gkey[0] = x0; c->gkey[1] = labels; c->gkey[2] = loss; c->gkey[3] = dx0;
    c->gkey_B = B; c->gkey_Bg = Bg; c->gkey_lr = lr;
    return DHEN_OK;   // this call's step already ran eagerly
  }
  CK(cudaGraphLaunch(c->gexec, st));
  g_launches += c->graph_launches;
  return DHEN_OK;
}

dhen_status dhen_params_io(dhen_ctx* c, int gi, float* host, int set, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_params_io: ctx is NULL");
  TuneScope ts_(&c->tune);
  if (gi < 0 || gi > c->cfg.n_layers) return fail(DHEN_E_SHAPE, "dhen_params_io: group=%d", gi);
  if (!host) return fail(DHEN_E_ALIGN, "dhen_params_io: host is NULL");
  Group& g = c->G[gi];
  cudaStream_t st = S(stream);
  const bool sh = c->dist.world > 1 && c->dist.fsdp;
  const int64_t lo = sh ? (int64_t)c->dist.rank * g.shard : 0;
  std::vector<float> pad;
  if (set) {
    to_internal(g, host, pad);
    CK(cudaMemcpyAsync(g.master, pad.data() + lo, (size_t)g.shard * 4, cudaMemcpyHostToDevice, st));
    CK(sgd_cast(g.master, nullptr, 0.f, g.comp, c->dt, g.shard, st));
    RET(fence_params(c, st));
    CK(cudaStreamSynchronize(st));
  } else {
    RET(gather_f32(c, g, g.master, pad, st));
    to_canonical(g, pad.data(), host);
  }
  return DHEN_OK;
}

dhen_status dhen_grads_get(dhen_ctx* c, int gi, float* host, void* stream) {
  if (!c) return fail(DHEN_E_STATE, "dhen_grads_get: ctx is NULL");
  TuneScope ts_(&c->tune);
  if (gi < 0 || gi > c->cfg.n_layers) return fail(DHEN_E_SHAPE, "dhen_grads_get: group=%d", gi);
  if (!host) return fail(DHEN_E_ALIGN, "dhen_grads_get: host is NULL");
  Group& g = c->G[gi];
  cudaStream_t st = S(stream);
  std::vector<float> pad;
  RET(gather_f32(c, g, c->dist.world > 1 ? g.gshard : g.grad, pad, st));
  to_canonical(g, pad.data(), host);
  return DHEN_OK;
}

}  // extern "C"
