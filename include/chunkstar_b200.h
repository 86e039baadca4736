/*
 * chunkstar_b200.h — C ABI of libchunkstar_b200.so, the B200 (sm_100a)
 * kernels behind the chunk-managed training step.
 *
 * The reference (`/root/reference/pkg/src/chunkstar`) has no FFI: its hot
 * path is a Python object API whose "kernels" are byte-accounting calls.
 * Each entry point below realises one of those accounting sites; the
 * Python engine (paper_2108_05818_b200.engine / .payload) calls them at
 * exactly the point the reference charges the bytes.
 *
 * Conventions
 *  - plain C types only; device pointers are void* / float*, sizes int64_t;
 *  - every GPU entry point takes a cudaStream_t (passed as void*) and is
 *    asynchronous; the library never allocates, frees or synchronises
 *    device memory (the caller owns all buffers) — except inside the NCCL
 *    communicator that cs_comm_init creates;
 *  - return 0 on success, a cudaError_t (>0) from the launch, or a
 *    negative CS_E* argument error; cs_last_error() describes the last
 *    failure on the calling thread;
 *  - dtype codes: CS_FP16 = 0, CS_BF16 = 1, CS_FP32 = 2 (sources only).
 *
 * Numerics (bit-identical in the CUDA kernels, the host kernel and the C
 * oracle; the association is torch.optim.Adam's CPU single-tensor path —
 * lerp/addcmul/addcdiv — with IEEE sqrt and division).  Scalars are formed
 * in double and rounded once: b2 = f(beta2), c1 = f(1-beta1),
 * c2 = f(1-beta2), decay = f(1 - lr*wd), wd, eps.  Per element, with
 * s = step scalars (CsStepState) and fma = fused multiply-add:
 *     g  = float(g16) * s.grad_scale
 *     if wd != 0:  adamw ? p = p * decay  :  g = fma(wd, p, g)
 *     m  = fma(c1, g - m, m)                      (lerp)
 *     v  = fma(c2 * g, g, v * b2)                 (mul_ + addcmul_)
 *     p  = p + ((-s.step_size) * m) / (sqrt(v) / s.sqrt_bc2 + eps)
 *     p16 = round_to_nearest_even(p)
 * When s.skip != 0 (non-finite gradients) p32 / m / v are not written and
 * p16 = round(p32): the 16-bit chunk held the step's gradients (grad
 * overwrite), so the unchanged parameters are put back over them.
 */
#ifndef CHUNKSTAR_B200_H
#define CHUNKSTAR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { CS_FP16 = 0, CS_BF16 = 1, CS_FP32 = 2 };

enum {
  CS_OK = 0,
  CS_EINVAL = -1,      /* bad argument (null pointer, negative count, dtype) */
  CS_EALIGN = -2,      /* a vectorised buffer is not 16-byte aligned */
  CS_ETOOMANY = -3,    /* work list longer than CS_MAX_ITEMS */
  CS_EUNAVAIL = -4,    /* NCCL could not be loaded (cs_comm_* / collectives) */
  CS_EINPROGRESS = -5  /* cs_comm_check: a nonblocking NCCL operation is pending */
};

#define CS_MAX_ITEMS 4096

/* Adam hyper-parameters (host struct, passed by pointer, copied at launch). */
typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
  int32_t adamw;           /* 1: decoupled weight decay (AdamW) */
} CsAdamHyper;

/* Per-step optimizer scalars; lives in DEVICE memory (64 bytes) and is
 * advanced on the device by cs_adam_prepare, so a step needs no host sync.
 * Initialise with cs_step_state_init. */
typedef struct {
  double  beta1_pow;       /* beta1^t after the last applied step */
  double  beta2_pow;
  int64_t step;            /* applied (non-skipped) steps */
  float   loss_scale;      /* dynamic loss scale used for THIS step's grads */
  int32_t good_steps;      /* consecutive finite steps since last growth */
  float   grad_scale;      /* out: (1/loss_scale) * clip_coef */
  float   step_size;       /* out: lr / (1 - beta1^t) */
  float   sqrt_bc2;        /* out: sqrt(1 - beta2^t) */
  int32_t skip;            /* out: 1 if the step is skipped (inf/nan) */
  float   grad_norm;       /* out: unscaled global L2 norm */
  float   sumsq;           /* in: global sum of squares of the scaled grads */
} CsStepState;

/* One fused-Adam work item: the used prefix [0, n) of one chunk position
 * (or of a non-chunked buffer such as the embedding).
 * p16: the fp16/bf16 chunk payload — holds the gradients on entry and the
 *      updated parameters on exit (grads reuse the param chunk, PAPER §4).
 * p32, m, v: the fp32 optimizer-state triplet of the same position. */
typedef struct {
  void*   p16;
  float*  p32;
  float*  m;
  float*  v;
  int64_t n;
} CsAdamItem;

/* One grad-reduction item: n elements of fp16/bf16 gradients. */
typedef struct {
  const void* g16;
  int64_t n;
} CsGradItem;

/* One pack / cast item: dst = chunk + offset (elements of dst dtype). */
typedef struct {
  void*       chunk;
  int64_t     offset;
  const void* src;
  int64_t     n;
} CsPackItem;

/* ---- library ------------------------------------------------------------ */
const char* cs_version(void);
const char* cs_last_error(void);
/* number of kernels this library has launched (process lifetime) */
int64_t     cs_launch_count(void);
/* number of SMs of the current device (grid sizing), or <0 on error */
int         cs_num_sms(void);
/* OpenMP team size the host kernels use for n_threads = requested:
 * requested if > 0, else (cores in this process's affinity mask) /
 * $LOCAL_WORLD_SIZE (one process per GPU shares the host with its local
 * peers; the division is skipped when CS_HOST_BOUND=1 says the mask is
 * already this rank's own share), at least 1.  Never omp_get_max_threads():
 * torchrun sets OMP_NUM_THREADS=1. */
int         cs_host_threads(int requested);

/* ---- K1: fused chunk Adam -------------------------------------------------
 * Replaces the accounting of Engine._adam_event for a GPU-placed position
 * (`/root/reference/pkg/src/chunkstar/engine.py:225-272`: charge_temp of one
 * fp32 staging chunk :227/:253, note_write of the triplet :254-255, param
 * release + place_payload :257-263).  One launch covers any number of
 * positions (grid-stride over all items, 128-bit loads/stores). */
int cs_adam_chunks(const CsAdamItem* items, int n_items, int dtype,
                   const CsAdamHyper* hyper, const CsStepState* d_state,
                   void* stream);
/* Tuning: select K1's data-movement variant (bit-identical results):
 * 0 SIMT register-tiled, 1 TMA-staged (cp.async.bulk + mbarrier ring with a
 * dedicated bulk-store warp; 5120-element tiles x 3 stages, 20 consumer
 * warps).  v < 0 only queries.  Default from $CS_ADAM_VARIANT, else 1.
 * Items whose pointers are not 16-byte aligned always run on variant 0.
 * The round-1 sweep of 25 tilings: profiles/r01/k1_variants.md. */
int cs_adam_variant(int v);

/* ---- K2: gradient sum of squares -------------------------------------------
 * Global grad-norm / found-inf for clipping and dynamic loss scaling (no
 * reference counterpart: the simulator has no numerics), in a canonical order
 * that does not depend on placement (HBM or host DRAM) or batching: each item
 * gets a double S_i defined tile by tile (specification in sumsq.cu, restated
 * by the C oracle); cs_grad_sumsq writes S_i into d_item_sums[slots[i]]
 * (slots NULL: i), cs_grad_sumsq_host computes the same S_i for items in host
 * memory, and cs_sumsq_finalize folds d_item_sums[0..n_slots) in slot order
 * (double) into d_state->sumsq.  d_scratch holds cs_sumsq_scratch(items)
 * floats (1/1024 of the gradient bytes). */
int64_t cs_sumsq_scratch(const CsGradItem* items, int n_items);
int cs_grad_sumsq(const CsGradItem* items, int n_items, int dtype, const int* slots,
                  float* d_scratch, int64_t scratch_elems, double* d_item_sums, void* stream);
int cs_sumsq_finalize(const double* d_item_sums, int n_slots, CsStepState* d_state,
                      void* stream);

/* ---- step scalars -------------------------------------------------------------
 * Device-side: consume d_state->sumsq, decide skip, clip coefficient,
 * bias corrections and the dynamic loss-scale update (growth/backoff). */
int cs_step_state_init(CsStepState* d_state, float init_loss_scale, void* stream);
int cs_adam_prepare(CsStepState* d_state, const CsAdamHyper* hyper,
                    float max_grad_norm, float growth_factor, float backoff_factor,
                    int32_t growth_interval, int32_t dynamic_scale, void* stream);

/* ---- K3 / K4: tensor -> chunk slot pack (grad overwrite / accumulate) -----
 * Realises the BWD grad overwrite of Engine._finish_compute_event
 * (`engine.py:177-190`: charge_temp(param_bytes), FINISH_BWD_GRAD_OVERWRITE,
 * note_write).  accumulate=0: slot = src (K3); 1: slot += src (K4).
 * Offsets need not be aligned (gap-free packing, `chunks.py:186-200`). */
int cs_pack(const CsPackItem* items, int n_items, int dtype, int accumulate,
            void* stream);

/* ---- K5: fp32 -> fp16/bf16 cast + pack -----------------------------------------
 * Materialises fp16 param chunks from fp32 init weights
 * (`chunks.py:297-314` init_on_cpu, `scenario.py:126`). src is fp32. */
int cs_cast_pack(const CsPackItem* items, int n_items, int dtype, void* stream);

/* ---- K6: optimizer-state birth ---------------------------------------------------
 * Lazy OS materialisation at the first ADAM on the planned device
 * (`engine.py:234-240`): p32 = float(src), m = v = 0.  src_dtype is
 * CS_FP16/CS_BF16 (widen the fp16 params) or CS_FP32 (copy master init). */
int cs_master_init(float* p32, float* m, float* v, const void* src, int src_dtype,
                   int64_t n, void* stream);

/* ---- host Adam for CPU-placed positions (PAPER §5 device-aware placement) ----
 * The placement plan may keep an optimizer triplet on the CPU
 * (`profiler.py:93-130`); the reference then moves grads D2H and new params
 * H2D as `adam_copy` (`engine.py:249-251, 265-267`).  This is the host
 * kernel that runs there (AVX2/F16C + OpenMP, same rounding as K1).
 * `state` is a HOST copy of the step scalars. Synchronous.
 * n_threads (here and in every host entry below): > 0 uses exactly that
 * many OpenMP threads; 0 uses cs_host_threads(0), this process's share of
 * the host cores. */
int cs_adam_chunks_host(const CsAdamItem* items, int n_items, int dtype,
                        const CsAdamHyper* hyper, const CsStepState* state,
                        int n_threads);

/* Out-of-place host Adam: in[i] = (gradients in p16, p32, m, v) are read,
 * out[i] = (p16, p32, m, v) receive the update (same bits as the in-place
 * call), with non-temporal stores when out is 32-byte aligned.  For the
 * speculative update of a CPU-placed position during the backward
 * (engine.py:249-267 bill it at ADAM): if the step overflows the inputs are
 * still intact.  in[i].n == out[i].n; state->skip must be 0. */
int cs_adam_chunks_host_oop(const CsAdamItem* in, const CsAdamItem* out, int n_items, int dtype,
                            const CsAdamHyper* hyper, const CsStepState* state, int n_threads);

/* Host twin of K2 for gradients in host DRAM (a chunk evicted to the CPU
 * before the ADAM event, CPU-placed positions, the CPU-placed embedding):
 * out[i] = S_i of items[i], bit-identical to what cs_grad_sumsq would write
 * for the same bytes in HBM. */
int cs_grad_sumsq_host(const CsGradItem* items, int n_items, int dtype, double* out,
                       int n_threads);

/* ---- host embedding operator (CPU-placed embedding) ----------------------------
 * PatrickStar's device-aware operator placement (PAPER §5): when the plan puts
 * the embedding on the CPU (`profiler.py:70-74` embedding_compute_device), its
 * fp16/bf16 weights stay in pinned host DRAM and only one activation block
 * crosses per pass (`engine.py:202-213`: B*S*H fp16 H2D at FWD, its gradient
 * D2H at BWD).  Host pointers; synchronous; AVX2/F16C + OpenMP.
 * fwd: out[i,:] = round(float(wte[tok[i],:]) + float(wpe[i % seq_len,:])).
 * bwd (grad overwrite, `engine.py:177-190`): gwte[v,:] = round(sum over tokens
 * i with tok[i]==v, ascending i, of float(dout[i,:])), 0 for rows no token hits;
 * gwpe[s,:] = round(sum over b ascending of float(dout[b*seq_len+s,:])).
 * gwte / gwpe may be the weight buffers themselves.  hidden % 8 == 0; every
 * token must lie in [0, vocab) (CS_EINVAL otherwise). */
int cs_embed_fwd_host(const int64_t* tokens, int64_t n_tokens, int seq_len, const void* wte,
                      const void* wpe, int64_t vocab, int hidden, void* out, int dtype,
                      int n_threads);
int cs_embed_bwd_host(const int64_t* tokens, int64_t n_tokens, int seq_len, const void* dout,
                      int64_t vocab, int hidden, void* gwte, void* gwpe, int dtype,
                      int n_threads, double* sumsq /* nullable: sum of squares of the
                      written gradients, double, row order (feeds the global norm) */);

/* ---- device embedding operator (GPU-placed embedding) ----------------------------
 * The GPU branch of the same placement decision (`engine.py:214-219`), with the
 * host operator's exact semantics (bit-identical results wherever it runs).
 * fwd: out[i,:] = round(float(wte[tok[i],:]) + float(wpe[i % seq_len,:])).
 * bwd: one kernel; `order` = token positions stably sorted by token id and
 * `row_start[v]..row_start[v+1]` = row v's range in it (V+1 entries, device);
 * writes every row of gwte [V,H] and gwpe [S,H] (fp32 sums in ascending token
 * order, one rounding); accumulate=1 adds the rounded row sums to gwte instead
 * (K4's slot += src, for a tied LM head whose dW was written there first).
 * Device pointers, 16-byte aligned buffers, stream-ordered.  Token ids are
 * device-resident and not validated on the host: a token outside [0, vocab)
 * reads nothing and its output row is NaN (so the loss is NaN and the
 * overflow check skips the step); the backward ignores such tokens. */
int cs_embed_fwd(const int64_t* tokens, int64_t n_tokens, int seq_len, const void* wte,
                 const void* wpe, int64_t vocab, int hidden, void* out, int dtype,
                 void* stream);
int cs_embed_bwd(const int64_t* order, const int64_t* row_start, int64_t n_tokens, int seq_len,
                 const void* dout, int64_t vocab, int hidden, void* gwte, void* gwpe,
                 int accumulate, int dtype, void* stream);

/* ---- fused LM-head cross entropy (the GPT step's loss) ----------------------
 * Forward: per-row loss = logsumexp(logits_row) - logits_row[target] and the
 * row's logsumexp, one pass over fp16/bf16 logits [rows, vocab].  Backward:
 * logits <- (softmax - onehot) * (*dloss) * scale, in place.  dloss is a
 * device scalar (the upstream gradient, e.g. the loss scale).  A target
 * outside [0, vocab) is never dereferenced: its row's loss and gradient are
 * NaN, so the loss reports it and the step's overflow check skips the update
 * (targets are device-resident and not validated on the host). */
int cs_xent_fwd(const void* logits, const int64_t* targets, int64_t rows, int64_t vocab,
                int dtype, float* loss_rows, float* lse_rows, void* stream);
int cs_xent_bwd(void* logits, const int64_t* targets, const float* lse_rows,
                const float* dloss, float scale, int64_t rows, int64_t vocab, int dtype,
                void* stream);

/* ---- non-affine LayerNorm (eps inside rsqrt), residual grad folded in -------
 * fwd: y = (x - mean) * rstd per row of [rows, H]; saves mean / rstd (fp32).
 * bwd: dx = rstd * (dy - mean(dy) - xhat * mean(dy * xhat)) + dres (dres nullable).
 * H must be 256 x {1,2,4,8,9,12,16} (cs_layernorm_supported). */
int cs_layernorm_supported(int H);
int cs_layernorm_fwd(const void* x, void* y, float* mean, float* rstd, int64_t rows, int H,
                     float eps, int dtype, void* stream);
int cs_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                     const void* dres, void* dx, int64_t rows, int H, int dtype, void* stream);

/* ---- MLP GEMMs with the GELU fused into the cuBLASLt epilogue --------------
 * mode 0 (forward):  out = gelu(x·Wᵀ), aux = x·Wᵀ      W [O,K], x [T,K] row-major
 * mode 1 (backward): out = (x·W) ⊙ gelu'(aux)          W [K,O], x = dy [T,K], aux [T,O]
 * gelu = tanh approximation.  workspace: caller-owned device buffer. */
int cs_gemm_gelu(int mode, const void* w, const void* x, void* out, void* aux, int64_t T,
                 int64_t O, int64_t K, int dtype, void* workspace, int64_t ws_bytes,
                 void* stream);

/* Residual GEMM, out = x·Wᵀ + res with the residual read by the GEMM (C ≠ D,
 * beta = 1): W [O,K], x [T,K], res / out [T,O] row-major; res is left intact. */
int cs_gemm_res(const void* w, const void* x, const void* res, void* out, int64_t T, int64_t O,
                int64_t K, int dtype, void* workspace, int64_t ws_bytes, void* stream);

/* ---- ZeRO chunk-group collectives (NCCL, loaded at first use) ---------------
 * For callers without torch.distributed (the Python executor uses
 * torch.distributed's NCCL by default; CS_COMM=native routes it here).
 * Protocol of `/root/reference/pkg/src/chunkstar/parallel.py:196-264`:
 * slot k of a p×count group buffer is rank k's chunk (position g·p+k,
 * `parallel.py:107-114`).  Comm calls return ncclResult_t (>0) on an NCCL
 * failure, CS_EUNAVAIL if libnccl.so.2 cannot be loaded.  Stream-ordered. */
#define CS_COMM_ID_BYTES 128
int cs_comm_version(void);                 /* NCCL_VERSION_CODE of the loaded NCCL */
int cs_comm_unique_id(void* id_out);       /* rank 0; share the 128 bytes out of band */
int cs_comm_init(const void* id, int nranks, int rank, void** comm);  /* current device */
int cs_comm_destroy(void* comm);
/* a18 (`parallel.py:196-223`): gather the group; in place when local is slot rank */
int cs_allgather(void* group_buf, const void* local, int64_t count, int dtype, void* comm,
                 void* stream);
/* a20 (`parallel.py:241-264`): local = mean over ranks of slot rank of group_buf */
int cs_reduce_scatter_avg(void* local, const void* group_buf, int64_t count, int dtype,
                          void* comm, void* stream);
/* replicated (non-chunked) grads: avg=1; the global sum of squares: avg=0, CS_FP32 */
int cs_allreduce(void* buf, int64_t count, int dtype, int avg, void* comm, void* stream);
/* Failure detection (surface NCCL async errors): 0 while the
 * communicator is healthy, CS_EINPROGRESS while a nonblocking operation is
 * pending, else the asynchronous ncclResult_t of a collective that failed
 * after it was enqueued (ncclCommGetAsyncError).  Poll while waiting. */
int cs_comm_check(void* comm);
/* ncclCommAbort: tear down without waiting for outstanding collectives
 * (unblocks kernels stuck on a dead peer); the handle is invalid after. */
int cs_comm_abort(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* CHUNKSTAR_B200_H */
