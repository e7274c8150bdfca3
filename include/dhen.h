/* dhen.h — C ABI of the B200-native DHEN layer-stack training path.
 *
 * DHEN (arXiv 2203.11014, "PAPER.md" = P:<line>): a stack of layers, each
 *   Y = Norm( Concat_i Interaction_i(X_n) + ShortCut(X_n) )          (Eq.(1))
 *   ShortCut(X_n) = X_n if len(X_n) == len(Y) else W_n^T X_n          (Eq.(2))
 * over the embedding list X_n (stored [B][m][d], row t = the paper's x^t),
 * with interaction modules Dot (Eq.(3)), SelfAttention (Eq.(4)), Conv (Eq.(5)),
 * Linear (Eq.(6)), DCN cross (Eq.(7), north-star DCN-v2 reading) and an MLP
 * single-tensor module.  Readings of silent passages: DESIGN.md §3.
 *
 * Memory ownership: the CALLER owns all device memory.  dhen_sizes() reports
 * how many bytes of `state` (parameters, master weights, gradients) and `work`
 * (saved activations + scratch, sized for batch_max_local) the library needs;
 * the caller allocates both (16-byte aligned; PyTorch in the Python binding)
 * and passes them to dhen_init(), which carves them.  They must outlive ctx.
 * Tensor arguments x/y/dy/dx/x0/dx0 are device pointers in the config's dtype
 * (fp32 or bf16), row-major [B][m][d], 16-byte aligned; labels/loss are fp32
 * device pointers.  Every call is stream-ordered on `stream` (a cudaStream_t;
 * NULL = legacy default stream) and returns before the GPU work finishes; the
 * caller keeps its buffers alive until the stream completes.
 *
 * Errors: every entry point returns a dhen_status.  A call that fails its
 * validation launches nothing (no partial updates).  dhen_last_error()
 * returns a thread-local message naming the call and the offending values.
 * Asynchronous CUDA faults surface as DHEN_E_CUDA on a later call.  No C++
 * exception crosses this boundary.  A ctx is used from one host thread.
 *
 * Collectives: with world > 1 the library owns an NCCL communicator (bootstrap
 * id from dhen_nccl_id() on rank 0, broadcast by the caller), shards every
 * parameter group across ranks (FSDP; on one host HSDP == FSDP,
 * P:171) and all ranks must make the same sequence of collective calls
 * (dhen_layer_fwd / dhen_layer_bwd / dhen_train_step).
 */
#ifndef DHEN_H_
#define DHEN_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dhen_ctx dhen_ctx;

typedef enum {
  DHEN_OK = 0,
  DHEN_E_CONFIG = 1,    /* invalid dhen_config / dhen_dist                      */
  DHEN_E_SHAPE = 2,     /* B out of range, bad layer / group index            */
  DHEN_E_ALIGN = 3,     /* a pointer not 16-byte aligned, or NULL             */
  DHEN_E_STATE = 4,     /* call out of order (bwd without fwd, ...)           */
  DHEN_E_CUDA = 5,      /* CUDA runtime / driver error                        */
  DHEN_E_NCCL = 6,      /* NCCL error                                          */
  DHEN_E_NONFINITE = 7, /* non-finite loss                             */
  DHEN_E_NOMEM = 8      /* caller buffers smaller than dhen_sizes() reported   */
} dhen_status;

/* Interaction module kinds. */
typedef enum {
  DHEN_DOT = 0,    /* Eq.(3): z = triu(X X^T) (strict, row-major pairs), U = reshape(W_m z, l, d)  */
  DHEN_ATTN = 1,   /* Eq.(4): U = W_u^T TransformerEncoderLayer(X) (post-norm, ReLU, no key bias)  */
  DHEN_CONV = 2,   /* Eq.(5): U = W_u^T ((1/C) sum_c K_c (*) X), same zero padding, no bias         */
  DHEN_DCN = 3,    /* Eq.(7) north star: T = X (.) (X W^T + b) + X per token, U = W_u^T T          */
  DHEN_LINEAR = 4, /* Eq.(6): U = W^T X on the token axis                                          */
  DHEN_MLP = 5,    /* U = reshape(W_m relu(W_2 relu(W_1 vec(X) + b_1) + b_2), l, d)           */
  DHEN_DCN_FULL = 7,/* flattened full-rank DCN-v2 (NEXT#3, R37): x = vec(X) in R^{m d}, A = x W^T + b with W in
                      R^{md x md}, T = x (.) A + x, U = W_u^T T (tokens)                                   */
  DHEN_DCN_LIT = 6 /* Eq.(7) read literally (NEXT#3, R31): per sample G = X_n X_n^T (d x d Gram over
                      tokens), u = G W + b, W in R^{d x l}, b in R^{l x d}; U[t][c] = (G W)[c][t] + b[t][c]  */
} dhen_kind;

typedef enum { DHEN_FP32 = 0, DHEN_BF16 = 1 } dhen_dtype;

typedef struct {
  int kind;          /* dhen_kind                                   */
  int l;             /* output token count l_i >= 1          */
  int heads;         /* ATTN: heads H, d % H == 0 (0 -> 2)          */
  int ffn_mult;      /* ATTN: FFN width = ffn_mult * d (0 -> 4)     */
  int conv_channels; /* CONV: C filters (0 -> 4)                    */
  int conv_k;        /* CONV: odd kernel extent k (0 -> 3)          */
  int mlp_hidden[2]; /* MLP: hidden widths (0 -> 1024)              */
} dhen_module;

typedef enum { DHEN_CONCAT = 0, DHEN_SUM = 1, DHEN_WSUM = 2 } dhen_ensemble;

typedef struct {
  int n_modules;
  const dhen_module* modules; /* in this order: concat offsets, canonical parameter order           */
  int ensemble;               /* a dhen_ensemble value -- P:91 "concatenation, sum, or weighted sum": CONCAT along
                                 tokens (R5, default); SUM or WSUM (one learnable scalar per module, R27,
                                 initialised to 1) of the modules' outputs, which then need equal l_i and
                                 give m_out = l                                                          */
  int dense_in;               /* 1: every module reads [X_n ; D] (m_in + dense_tokens tokens), D = the first
                                 dhen_config.dense_tokens tokens of X_0 -- P:64 "the raw numerical (dense)
                                 features can be part of the input to any modules ... in every layer" (NEXT#3,
                                 R38); the shortcut and the LayerNorm still see X_n                         */
} dhen_layer;

typedef struct {
  int m0;                 /* input token count m of X_0             */
  int d;                  /* embedding dim, d % 8 == 0                      */
  int n_layers;
  const dhen_layer* layers;
  int dtype;              /* dhen_dtype: storage / compute-operand dtype    */
  float ln_eps;           /* LayerNorm epsilon (0 -> 1e-5)                  */
  int batch_max_local;    /* largest per-rank B any call will use          */
  unsigned long long seed;/* parameter init seed                            */
  int optimizer;          /* 0: SGD theta -= lr g (R18, default); 1: Adam (P:158's optimizer, NEXT#3): fp32
                             moments on the master shard, PyTorch semantics, no weight decay; 2: the same
                             Adam with its moments stored in bf16 ("BF16 optimizer", R35: fp32 math,
                             RNE storage, half the optimizer-state memory)                                  */
  float adam_beta1, adam_beta2, adam_eps;   /* Adam (0 -> 0.9, 0.999, 1e-8)                          */
  int dense_tokens;       /* R38: X_0[:, :dense_tokens] are the dense tokens D injected into dense_in layers
                             (0: none); dL/dX_0 of those tokens adds every injected layer's dD             */
  int recompute;          /* activation recompute ("activation checkpointing", NEXT#2), bit mask:
                             1 = the attention FFN hidden F (and its ReLU bitmask) is not kept from forward
                             to backward: one shared buffer, F recomputed by the backward (one FFN1 GEMM per
                             layer; at C4 16 GB less work memory); results are bit-identical            */
} dhen_config;

typedef struct {
  int rank, world;              /* world == 1: no collectives                   */
  unsigned char nccl_id[128];   /* backend 0: ncclUniqueId from rank 0 (world > 1); backend 1: dhen_loopback_id() */
  int fsdp;                     /* 1: fully sharded (default); 0: replicated DP */
  int backend;                  /* 0: NCCL (one process per GPU, the product path); 1: loopback -- `world` virtual
                                   ranks in ONE process on one GPU, one host thread and ctx per rank, collectives
                                   = host rendezvous + stream/event-ordered copies and fixed-order sums (a test
                                   backend for the FSDP path on a one-GPU machine; no CUDA-graph capture) */
  int grad_bf16;                /* 1: gradients reduce-scattered in bf16 (the paper's quantized collectives,
                                   P:158 / P:277: cast, bf16 sum, widened into the fp32 gradient shard); 0: fp32 */
} dhen_dist;

/* Host-only, pure: validates a config (preconditions S:186, S:195, S:204,
 * l >= 1, d % 8 == 0, d % heads == 0).  DHEN_E_CONFIG with a message. */
dhen_status dhen_validate(const dhen_config* cfg);

/* Host-only: bytes of caller-provided `state` and `work` device memory. */
dhen_status dhen_sizes(const dhen_config* cfg, const dhen_dist* dist,
                       size_t* state_bytes, size_t* work_bytes);

/* Host-only: total / per-rank-shard element counts of parameter group g
 * (g in [0, n_layers) = layer g, g == n_layers = head).  Canonical order:
 * DESIGN.md §2 table. */
dhen_status dhen_group_numel(const dhen_config* cfg, const dhen_dist* dist, int group,
                             size_t* numel, size_t* shard_numel);

/* Rank 0: a fresh NCCL unique id (128 bytes) to broadcast to the other ranks. */
dhen_status dhen_nccl_id(unsigned char out[128]);

/* A fresh loopback-group id (dhen_dist.backend = 1): every virtual rank of the group passes the same id. */
dhen_status dhen_loopback_id(unsigned char out[128]);

/* Bytes this rank's collectives have moved since init (ring convention: an all-gather of n elements per rank
 * receives (world - 1) n, a reduce-scatter to n per rank sends (world - 1) n, fp32 = 4 B, bf16 = 2 B).  One
 * FSDP training step moves (world - 1) / world x (2 x 2 B per gathered copy + 4 B) per padded parameter
 * (DESIGN.md §10 gives the exact per-step formula).  0 when world == 1. */
unsigned long long dhen_comm_bytes(const dhen_ctx* ctx);

/* Carve state/work, initialise parameters from cfg->seed (U(+-1/sqrt(fan_in)),
 * LN gamma = 1, beta = 0), create the NCCL communicator when world > 1 (a
 * collective over all ranks).  Launches on `stream`. */
dhen_status dhen_init(const dhen_config* cfg, const dhen_dist* dist, void* state, size_t state_bytes,
                      void* work, size_t work_bytes, void* stream, dhen_ctx** out);

/* Forward of layer n: x [B][m_in][d] -> y [B][m_out][d] (Eq.(1)(2)).  Saves
 * the activations layer n's backward needs (x is referenced, not copied: keep
 * it unchanged until dhen_layer_bwd(n) returns).  Collective when world > 1. */
dhen_status dhen_layer_fwd(dhen_ctx* ctx, int layer, const void* x, void* y, int B, void* stream);

/* Backward of layer n given dy [B][m_out][d]: accumulates (+=) the layer's
 * parameter gradients and writes dx [B][m_in][d] (dx may be NULL).
 * Requires a preceding dhen_layer_fwd(n) with the same B (else DHEN_E_STATE).
 * With world > 1, gradients are reduce-scattered to the owner shards. */
dhen_status dhen_layer_bwd(dhen_ctx* ctx, int layer, const void* dy, void* dx, int B, void* stream);

/* One training step on the local batch x0 [B][m0][d], labels [B] (0/1 fp32):
 * zero grads, forward all layers, head z_b = w_h . mean_t Y_N[b,t] + b_h,
 * loss = sum_b BCEWithLogits(z_b, y_b) / B_global (R17, R21), backward,
 * reduce-scatter (world > 1), then the optimizer on the fp32 masters: SGD theta -= lr * g (R18), or Adam
 * (cfg->optimizer = 1; its step count lives on the device, so graph replays stay correct).
 * loss_dev (nullable, fp32 device scalar) receives the loss of this rank's
 * samples (sum over ranks = global loss).  dx0 (nullable) receives dL/dx0. */
dhen_status dhen_train_step(dhen_ctx* ctx, const void* x0, const float* labels, int B, int B_global,
                            float lr, float* loss_dev, void* dx0, void* stream);

/* dhen_train_step through a CUDA graph: the first call with a given argument set runs the step
 * eagerly and captures it; later calls with the same (x0, labels, B, B_global, lr, loss_dev, dx0)
 * replay the graph (one cudaGraphLaunch on `stream`).  Buffer contents may change between calls,
 * pointers may not (a change re-captures).  world > 1 or profiling: plain dhen_train_step. */
dhen_status dhen_train_step_graphed(dhen_ctx* ctx, const void* x0, const float* labels, int B, int B_global,
                                    float lr, float* loss_dev, void* dx0, void* stream);

/* One training step from HOST buffers (the end-to-end path a data loader drives): x0_host [B][m0][d] (dtype) and
 * labels_host [B] fp32 (page-locked memory, e.g. cudaHostAlloc, for asynchronous copies) are copied host -> device
 * on the context's copy stream into one of two staging slots (call k uses slot k % 2; its upload waits only for
 * call k - 2's step to have consumed that slot, so an upload overlaps the previous step), moved into the step's
 * input buffers on `stream`, the step runs (dhen_train_step_graphed semantics), and this rank's loss is copied
 * device -> host into *loss_host.  sync = 1: `stream` is synchronised before returning (*loss_host valid); sync = 0:
 * *loss_host becomes valid, and x0_host / labels_host may be reused, once `stream` has been synchronised.
 * Device buffers are allocated on the first call (2 x B_max staging + inputs). */
dhen_status dhen_train_step_host(dhen_ctx* ctx, const void* x0_host, const float* labels_host, int B, int B_global,
                                 float lr, float* loss_host, int sync, void* stream);

/* Forward of the whole stack + head without backward: logits_dev [B] fp32. */
dhen_status dhen_forward(dhen_ctx* ctx, const void* x0, int B, float* logits_dev, void* stream);

dhen_status dhen_zero_grad(dhen_ctx* ctx, void* stream);

/* Canonical fp32 parameters of group g: set == 1 copies host -> master
 * weights (and refreshes the compute copy), set == 0 copies masters -> host.
 * `host` holds dhen_group_numel() floats.  Synchronises `stream`. */
dhen_status dhen_params_io(dhen_ctx* ctx, int group, float* host, int set, void* stream);

/* Accumulated fp32 gradients of group g (reduced over ranks when world > 1)
 * -> host.  Synchronises `stream`. */
dhen_status dhen_grads_get(dhen_ctx* ctx, int group, float* host, void* stream);

/* Per-op device timing: enable != 0 clears and starts recording a CUDA event
 * pair around every op the library launches (on the op's stream); 0 stops.
 * enable == 1 serialises the side stream onto the layer stream (every op's time is its own);
 * enable == 2 keeps the concurrency (the timeline of dhen_debug_profile_trace shows it).
 * Adds two event records per op: for measurement passes, not the timed step. */
dhen_status dhen_profile(dhen_ctx* ctx, int enable);

typedef struct {
  char name[40];                /* op tag, e.g. "dot.proj", "layer.ln"           */
  unsigned long long launches;  /* recorded launches of this op                   */
  double ms;                    /* summed device time (CUDA events)               */
  double flops;                 /* summed algorithmic FLOPs (2 M N K per GEMM)    */
  double bytes;                 /* summed algorithmic HBM bytes (operands once)   */
  unsigned long long tc_launches; /* launches that ran on the tcgen05 tensor-core path */
} dhen_op_stat;

/* Aggregate the recorded ops by tag (synchronises on the recorded events):
 * writes min(cap, *n) entries to out, *n = number of distinct tags. */
dhen_status dhen_profile_read(dhen_ctx* ctx, dhen_op_stat* out, int cap, int* n);

/* Number of library kernels launched since init (a host-side counter). */
unsigned long long dhen_launch_count(const dhen_ctx* ctx);

const char* dhen_last_error(void);
void dhen_destroy(dhen_ctx* ctx);

/* ---------------------------------------------------------------------------------------------------------
 * Feature processing layer (NEXT#4; "we use the same feature processing layer in DLRM"; readings
 * R32-R34): the step in front of the stack that produces X0 [B][m0][d], m0 = n_dtok + n_sparse:
 *   X0[b][0 .. n_dtok)        = the bottom MLP of the numerical features, H_k = relu(H_{k-1} W_k^T + b_k),
 *                               H_0 = dense[b], output width n_dtok * d read as n_dtok tokens (R32);
 *   X0[b][n_dtok + t]         = sum of the rows of table t (R_t x d) listed in bag (b, t)  (sum pooling).
 * Tables are fp32 (lookups and sums in fp32, X0 stored in `dtype`); W_k [out][in] / b_k have fp32 masters
 * and `dtype` compute copies.  One object owns its device memory (cudaMalloc at init, freed by destroy).
 * --------------------------------------------------------------------------------------------------------- */
typedef struct {
  int n_sparse;             /* sparse features = tables, one pooled token each (>= 0)                      */
  const long long* rows;    /* [n_sparse] table rows R_t (host)                                             */
  int n_dense;              /* numerical features per sample                                               */
  int n_hidden;             /* bottom-MLP hidden layers                                                     */
  const int* hidden;        /* [n_hidden] hidden widths (host)                                              */
  int n_dtok;               /* dense tokens (0: no bottom MLP)                                              */
  int d;                    /* token dimension: 4 | d, d <= 512                                             */
  int dtype;                /* dhen_dtype of dense, X0 and dX0                                              */
  int max_batch;            /* largest B of a forward                                                       */
  long long max_nnz;        /* largest total number of ids of a forward (<= 2^31 - 1)                        */
  unsigned long long seed;  /* init: tables U(+-sqrt(1/R_t)), W_k / b_k U(+-1/sqrt(fan_in))                 */
} dhen_fp_config;
typedef struct dhen_fp dhen_fp;

/* Allocate and initialise (synchronises `stream`).  DHEN_E_CONFIG on an invalid config, DHEN_E_NOMEM when
 * the device allocation fails. */
dhen_status dhen_fp_init(const dhen_fp_config* cfg, void* stream, dhen_fp** out);

/* Sharded feature processing (NEXT#4, reading R36): `dist->world` ranks train data-parallel on B samples
 * each (global sample k B + b = rank k's sample b).  Every table is cut into S_t equal column shards and the shards
 * are placed on ranks by LPT (dhen_fp_shard_plan; the same plan on every rank); a rank stores only its shards and
 * the whole bottom MLP (data parallel).  Collective over the ranks (dist->backend: NCCL or loopback, as for the
 * stack).  Forward: `ids` / `offsets` / `nnz` describe the GLOBAL batch's bags of the tables this rank owns a shard
 * of (dhen_fp_owned_tables, ascending; bag (k B + b, j) = ids[offsets[(k B + b) n_owned + j] ..]) -- the input
 * pipeline routes the sparse features, as DLRM data loaders do -- and `dense` this rank's B samples; the rank pools
 * its shards for all world x B samples, one pooled all-to-all moves every block to its samples' rank, and X0
 * [B][m0][d] is assembled there.  Backward: the reverse all-to-all gives every shard owner dX0's columns of its
 * shards, its rows take the sorted-run SGD, and the bottom MLP's gradients are all-reduced (sum, rank order).
 * world = 1 (or dist = NULL) is dhen_fp_init. */
dhen_status dhen_fp_init_dist(const dhen_fp_config* cfg, const dhen_dist* dist, void* stream, dhen_fp** out);
/* The tables this rank owns a shard of (ascending) -> tables[] (nullable: count only); returns their count. */
int dhen_fp_owned_tables(const dhen_fp* fp, int* tables);
/* The column-shard plan for `world` ranks: shards[t] = S_t (a power of two: a shard's elements at most half of one
 * rank's share of all table elements, >= 32 columns each); owner[] = the rank of each shard, tables in order and
 * shards of a table in column order (sum_t S_t entries).  LPT: largest R_t d / S_t first onto the least-loaded rank. */
dhen_status dhen_fp_shard_plan(const dhen_fp_config* cfg, int world, int* shards, int* owner);

/* Forward of B samples (device pointers): ids int32 [nnz] (each relative to its table), offsets int32
 * [B n_sparse + 1] with bag (b, t) = ids[offsets[b n_sparse + t] .. offsets[b n_sparse + t + 1]) (empty bags
 * pool to 0), dense [B][n_dense] in dtype (16-B aligned; ignored when n_dtok = 0), x0 [B][m0][d] out (16-B
 * aligned).  ids outside [0, R_t) are skipped and counted (dhen_fp_bad_ids).  ids, offsets, dense and x0 are
 * referenced by the following dhen_fp_backward_sgd: keep them unchanged until it returns. */
dhen_status dhen_fp_forward(dhen_fp* fp, const int* ids, const int* offsets, long long nnz, const void* dense, int B,
                            void* x0, void* stream);

/* Backward of the last forward given dx0 [B][m0][d] (dtype; e.g. dhen_train_step's dx0), fused with SGD:
 * E_t[r] -= lr * sum over r's occurrences of dx0[b][n_dtok + t] (rows summed in sample order, deterministic;
 * untouched rows unchanged, R34), then W_k, b_k -= lr * their gradients (fp32 masters, copies refreshed). */
dhen_status dhen_fp_backward_sgd(dhen_fp* fp, const void* dx0, float lr, void* stream);

/* Parameter `which` as fp32 on the host: 0 .. n_sparse-1 table t [R_t][d] (sharded: only this rank's column
 * shards of it are read / written; other columns of `host` are left as they are); then W_1, b_1, W_2, b_2, ...
 * (W_k [out][in]).  set = 1 writes (and refreshes the compute copy), 0 reads.  Synchronises `stream`. */
dhen_status dhen_fp_params_io(dhen_fp* fp, int which, float* host, int set, void* stream);
/* Elements of parameter `which` (-1 on an invalid config / index). */
long long dhen_fp_param_numel(const dhen_fp_config* cfg, int which);
/* ids skipped as out of range since init (synchronous read). */
long long dhen_fp_bad_ids(dhen_fp* fp);
void dhen_fp_destroy(dhen_fp* fp);

#ifdef __cplusplus
}
#endif
#endif /* DHEN_H_ */
