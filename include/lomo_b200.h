/*
 * lomo_b200.h -- C-ABI of the B200 (sm_100a) LOMO fused-update hot path.
 *
 * This is the drop-in boundary for the per-parameter hook body of the
 * reference `fusedtrain` (CPU/numpy, /root/reference/pkg/src/fusedtrain):
 *
 *   reference (file:line)                               replaced by
 *   --------------------------------------------------  --------------------------
 *   optim.py:52-54   apply_update(param, g, lr)          lomo_fused_update  (K1)
 *   tensor.py:74-81  Tensor.assign (write-back)          K1 store (RNE to dtype)
 *   tensor.py:30-38  round_through_half                  K1 store (cvt.rn.f16.*)
 *   optim.py:126-128 LOMO hook (update, CONSUME)         K1, state=NULL-equivalent
 *   stabilize.py:82-86,168-173 clip_by_value in hook     K1 clip_value > 0
 *   stabilize.py:193-200 probe_hook (overflow, sumsq)    lomo_probe         (K2)
 *   stabilize.py:204-213 norm / clip-coef decision       lomo_finalize_norm (K3a)
 *   stabilize.py:155-159 _skip -> LossScaler.on_overflow K3a (on device)
 *   stabilize.py:115-127 LossScaler.on_overflow/on_clean K3a / lomo_scaler_on_clean (K3b)
 *   stabilize.py:217-224 update_hook (unscale,clip,coef) K1 with LOMO_USE_SCALE|LOMO_USE_COEF
 *   optim.py:63-65   _require_finite(loss)               lomo_begin_step (device flag)
 *   tape.py:330-405  Tape.backward/_deliver hook call    torch post-accumulate-grad hook
 *                                                         (host side)
 *
 * Conventions
 *   - Every entry point is asynchronous on `stream` (a cudaStream_t passed as
 *     void*), never synchronises the host, never allocates, and returns 0 on
 *     success or a positive cudaError_t / negative LOMO_E* code.  No C++
 *     exception crosses this boundary.
 *   - `p` and `g` are device pointers to `n` contiguous elements of `dtype`.
 *     The update is in place on `p`; `g` is read once.  Any alignment works;
 *     16-byte-aligned p/g with equal misalignment take the 128-bit path.
 *   - The device-resident step state (`lomo_state` + per-slot sum-of-squares
 *     partials + K2 scratch) is one block of lomo_state_bytes(nslots) bytes
 *     owned by the caller (allocated with the framework's allocator).
 */
#ifndef LOMO_B200_H
#define LOMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOMO_ABI_VERSION 2 /* 2: the pass-2 record at offset 128 moved sumsq[] to 160; LOMO_CHAINED */

/* storage dtype of p and g (reference: Precision, tensor.py:19-21;
 * FULL == float64 storage, HALF_EMULATED == binary16; bf16 is new). */
typedef enum {
  LOMO_F32 = 0,
  LOMO_F16 = 1,
  LOMO_BF16 = 2,
  LOMO_F64 = 3
} lomo_dtype;

/* arithmetic width of the update.  F64 reproduces the reference's full-width
 * arithmetic (optim.py:9-13) and rounds f64 -> storage directly (bit-exact with
 * numpy's float64 -> float16 cast); F32 is the fp32-math hot path. */
typedef enum {
  LOMO_MATH_F32 = 0,
  LOMO_MATH_F64 = 1
} lomo_math;

/* flags for lomo_fused_update / lomo_probe */
#define LOMO_USE_SCALE 0x1u /* g *= state->inv_scale  (stabilize.py:218)           */
#define LOMO_USE_COEF 0x2u  /* g *= state->clip_coef  (stabilize.py:221-222)       */
#define LOMO_USE_SKIP 0x4u  /* no-op when state->skip (stabilize.py:204-205,       */
                            /*                          optim.py:63-65)            */
#define LOMO_LR_FROM_STATE 0x10u /* K1: lr = state->lr (set by lomo_set_lr), so a  */
                                 /* CUDA graph of the step needs no re-capture when */
                                 /* the schedule changes lr                         */
#define LOMO_DEFER_ROWS 0x20u /* K6: leave the partial sums in the workspace; */
                              /* lomo_gemm_probe_finish reduces a batch of them  */
#define LOMO_PROBE_KEEP_GRAD 0x40u /* K6: grad_out receives dW in the storage  */
                                   /* dtype (else a 16-byte scratch)           */
#define LOMO_CHAINED 0x80u /* K1 / K2: the kernel launched just before this one */
                           /* on the stream is a K1 (or K1 multi) -- for K2 a K2 */
                           /* (or K2 multi) on another slot -- on OTHER tensors, */
                           /* as in a run of updates over kept or replayed       */
                           /* gradients; the kernel then loads and stores before */
                           /* the PDL wait and waits only at its end, overlapping */
                           /* the previous launch's drain.  UNSAFE when the      */
                           /* previous kernel writes this p or g (e.g. the same  */
                           /* tensor twice in a row) or is a producer that       */
                           /* triggers its dependents before its writes complete. */
#define LOMO_ACCUM_F64 0x8u /* K2: accumulate every square in f64 (the reference's */
                            /* float64 dot, stabilize.py:199); default for 16-bit   */
                            /* storage: exact fp32 squares summed per 16-byte      */
                            /* vector in fp32, vectors accumulated in f64           */

#define LOMO_E_ARG (-1)     /* invalid argument (null pointer, n < 0, bad dtype)   */
#define LOMO_E_SLOT (-2)    /* slot outside [0, nslots)                            */

/* Device-resident step state.  Layout is part of the ABI (host code may view
 * individual fields, e.g. `scale` to multiply the loss on device). */
typedef struct lomo_state {
  double scale;          /*   0: dynamic loss scale, power of two (stabilize.py:106) */
  double inv_scale;      /*   8: 1/(scale*grad_div), the factor K1/K2 apply to g       */
  double min_scale;      /*  16                                                      */
  double max_scale;      /*  24                                                      */
  double clip_coef;      /*  32: min(1, max_norm/N) or 1 (stabilize.py:212-213)      */
  double total_norm;     /*  40: N of the last finalize                              */
  double sumsq_total;    /*  48: sum over slots, in slot order                       */
  double max_norm;       /*  56: config (<= 0: no norm clip)                         */
  int32_t growth_interval; /* 64                                                     */
  int32_t clean_steps;   /*  68: stabilize.py:110                                    */
  int32_t overflow;      /*  72: non-finite grad (K2) or loss (begin_step) seen      */
  int32_t skip;          /*  76: this step is dropped; K1 with LOMO_USE_SKIP no-ops  */
  int32_t underflow;     /*  80: on_overflow would go below min_scale (fatal)        */
  int32_t nslots;        /*  84                                                      */
  int32_t steps_applied; /*  88                                                      */
  int32_t steps_skipped; /*  92                                                      */
  uint32_t ticket;       /*  96: K2 last-block ticket (internal)                     */
  int32_t has_scaler;    /* 100                                                      */
  float scale_f32;       /* 104: scale as fp32 (exact: power of two), for loss*scale */
  int32_t error;         /* 108: sticky; 1: a probe kernel got slot >= nslots;   */
                         /*      2: a peer barrier timed out (sharded K4)        */
  double grad_div;       /* 112: data-parallel gradient divisor (world size; 1)      */
  double lr;             /* 120: learning rate read under LOMO_LR_FROM_STATE          */
  /* followed by: 32 bytes at offset 128: the pass-2 record {int32 skip; float
   *              inv_scale, clip_coef, lr} (fp32 copies the state kernels
   *              republish whenever they change a field; the fp32-math K1
   *              reads it with one 16-byte load, internal);
   *              double  sumsq[nslots];  at LOMO_STATE_SLOTS_OFFSET (per-slot totals)
   *              int32_t nblocks[nslots], padded to 8 bytes;  (K2 CTAs per slot)
   *              double  partials[nslots][LOMO_PROBE_BLOCKS_PER_SLOT];
   * K2 writes one partial per CTA (no atomics); K3a reduces each row in CTA
   * order, then the slots in slot order: deterministic. */
} lomo_state;

#define LOMO_PROBE_BLOCKS_PER_SLOT 8192
#define LOMO_STATE_SLOTS_OFFSET 160 /* sizeof(lomo_state) + the 32-byte pass-2 record */

/* 128-byte host snapshot of the state header (lomo_read_status). */
typedef lomo_state lomo_status;

/* ---- library / state management ------------------------------------- */
int lomo_abi_version(void);
size_t lomo_state_bytes(int nslots);
/* Initialise a state block (device memory).  scale <= 0 => no loss scaler
 * (scale = 1).  max_norm <= 0 => no global-norm clip.  grad_div <= 0 => 1; in
 * sharded data-parallel mode it is the world size, so LOMO_USE_SCALE turns the
 * reduce-scattered SUM of per-rank mean gradients into the global mean. */
int lomo_state_init(void* state, int nslots, double scale, int growth_interval,
                    double min_scale, double max_scale, double max_norm,
                    double grad_div, void* stream);
/* Start of a step: clear overflow/skip/underflow and the slot partials; if
 * `loss` is non-NULL, set overflow+skip when it is non-finite
 * (optim.py:63-65 / stabilize.py:185-189). */
int lomo_begin_step(void* state, const void* loss, int loss_dtype, void* stream);
/* Copy the 128-byte header to host memory `out` (async on `stream`; the
 * caller synchronises before reading -- the one host sync per step). */
int lomo_read_status(const void* state, lomo_status* out, void* stream);

/* ---- K1: fused update ------------------------------------------------ */
/* p <- round_dtype(p*(1-lr*wd) - lr * coef * clip(g * inv_scale, +-clip_value))
 *   clip_value <= 0 : no value clip;  weight_decay == 0 : reference semantics
 *   (the reference LOMO has no weight decay, optim.py:52-54). */
int lomo_fused_update(void* p, const void* g, int64_t n, int dtype, int math,
                      double lr, double clip_value, double weight_decay,
                      unsigned flags, const void* state, void* stream);

/* Multi-tensor K1: one launch per 64 (p, g, n) triples.  The three lists are
 * HOST arrays (they are packed into the kernel's parameter block); used to
 * coalesce the many tiny tensors (norm scales) of a backward pass. */
int lomo_fused_update_multi(void* const* p_list, const void* const* g_list,
                            const int64_t* n_list, int count, int dtype, int math,
                            double lr, double clip_value, double weight_decay,
                            unsigned flags, const void* state, void* stream);

/* Set state->lr (a one-thread kernel; launch it outside a captured graph). */
int lomo_set_lr(void* state, double lr, void* stream);
/* Restore the LossScaler's live state from a checkpoint (stabilize.py:94-127:
 * scale -- a power of two -- and clean_steps) and the applied / skipped step
 * counters; 1/scale, the fp32 scale and the pass-2 record follow.  The scale
 * is ignored for a state block initialised without a scaler. */
int lomo_set_scaler_state(void* state, double scale, int clean_steps, int steps_applied,
                          int steps_skipped, void* stream);

/* ---- K2: probe (two-pass pass 1) --------------------------------------- */
/* sumsq[slot] = sum((g * inv_scale)^2) (deterministic: fixed-order f64 tree);
 * state->overflow |= any(!isfinite(g)).  flags: LOMO_USE_SCALE. */
int lomo_probe(const void* g, int64_t n, int dtype, int slot, unsigned flags,
               void* state, void* stream);

/* Multi-tensor K2 for small tensors: one CTA per tensor writes sumsq[slot]
 * directly (host arrays, as for lomo_fused_update_multi). */
int lomo_probe_multi(const void* const* g_list, const int64_t* n_list,
                     const int* slot_list, int count, int dtype, unsigned flags,
                     void* state, void* stream);

/* ---- K3: finalisers (single CTA) --------------------------------------- */
/* K3a: total = sum(sumsq[0..nslots)) in slot order; N = sqrt(total);
 * skip = overflow || (max_norm > 0 && !isfinite(N)); coef per
 * stabilize.py:209-213; on skip, LossScaler.on_overflow on device. */
int lomo_finalize_norm(void* state, void* stream);
/* K3b: LossScaler.on_clean on device when the step was applied. */
int lomo_scaler_on_clean(void* state, void* stream);
/* Sharded mode (ZeRO-3 shards, one rank per GPU):
 * lomo_local_norm_partial writes {sum(sumsq slots in slot order), overflow}
 * of THIS rank into out2_dev[0..1] (it is what the all-gather exchanges);
 * lomo_finalize_norm_ranks takes the gathered [world][2] rows and runs K3a's
 * decision on the rank-ordered sum (deterministic across ranks). */
int lomo_local_norm_partial(const void* state, double* out2_dev, void* stream);
int lomo_finalize_norm_ranks(void* state, const double* parts_dev, int world,
                             void* stream);

/* ---- K4: reduce-scatter fused with the update (sharded mode) ---------- */
/* Every rank's flat bucket gradient lives in symmetric (peer-mapped) memory;
 * peer_bufs_dev is a DEVICE array of the `world` (<= 16) peer base pointers.
 * Rank r owns elements [offset, offset+n) of the bucket: K4 loads that slice
 * from every peer over NVLink, sums in rank order (deterministic) and applies
 * the K1 update to p_shard (n elements) -- or, for the probe, the K2 sum of
 * squares into `slot` -- without writing the reduced gradient anywhere.
 * offset*sizeof(dtype) and n*sizeof(dtype) must be multiples of 16.
 * Replaces NCCL reduce_scatter + K1/K2. */
int lomo_fused_rs_update(void* p_shard, const void* const* peer_bufs_dev, int world,
                         int64_t offset, int64_t n, int dtype, int math, double lr,
                         double clip_value, double weight_decay, unsigned flags,
                         const void* state, void* stream);
int lomo_fused_rs_probe(const void* const* peer_bufs_dev, int world, int64_t offset,
                        int64_t n, int dtype, int slot, unsigned flags, void* state,
                        void* stream);
/* K4 probe that also KEEPS the reduced slice: `out` (n elements of `dtype`,
 * 16-byte aligned) receives the rank-ordered sum rounded to the storage dtype
 * -- what a reduce-scatter would have written -- and the squares are taken of
 * those rounded values.  Pass 2 then updates from `out` with K1 (ShardedLOMO
 * keep_grads over K4: no second reduction).  probe_hook stabilize.py:193-200
 * on the reduced gradient. */
int lomo_fused_rs_probe_keep(const void* const* peer_bufs_dev, int world, int64_t offset,
                             int64_t n, int dtype, int slot, unsigned flags, void* state,
                             void* out, void* stream);
/* NVLS form of K4: `mc` is this rank's slice [offset, offset+n) of the bucket
 * at a MULTICAST address (lomo_mc_bind); every 16-byte vector is fetched with
 * multimem.ld_reduce.add (the NVSwitch sums the `world` copies in flight, fp32
 * accumulation for 16-bit storage, one rounding to the storage dtype -- what
 * an NCCL reduce-scatter would deliver) and fed to the K1 arithmetic / the K2
 * sum of squares.  dtype F32, F16 or BF16; n*sizeof(dtype) and the address
 * 16-byte aligned. */
int lomo_fused_mc_update(void* p_shard, const void* mc, int64_t n, int dtype, int math, double lr,
                         double clip_value, double weight_decay, unsigned flags,
                         const void* state, void* stream);
int lomo_fused_mc_probe(const void* mc, int64_t n, int dtype, int slot, unsigned flags,
                        void* state, void* stream);
/* NVLS form of lomo_fused_rs_probe_keep: `out` receives the switch's sum
 * (already rounded to the storage dtype by multimem.ld_reduce). */
int lomo_fused_mc_probe_keep(const void* mc, int64_t n, int dtype, int slot, unsigned flags,
                             void* state, void* out, void* stream);

/* ---- peer memory for K4 (transport; one process per GPU) --------------- */
/* The reduce-over-peers kernels need the ranks' bucket buffers mapped into
 * each other's address space and a device-side barrier between ranks.  Two
 * transports, both set up once per optimizer (host calls, synchronous):
 *
 * (1) CUDA IPC (any CUDA peers: NVLink P2P, or two processes sharing one GPU).
 *     lomo_ipc_alloc: cudaMalloc(bytes) zero-filled + its IPC handle
 *     (lomo_ipc_handle_bytes() bytes, copied to handle_out) -- the buffers
 *     and a signal area live in this one allocation; lomo_ipc_open maps a
 *     peer's handle (lazy peer access), lomo_ipc_close unmaps it,
 *     lomo_ipc_free frees an own allocation.
 * (2) NVLS multicast (NVSwitch; lomo_mc_supported() == 1).  Rank 0 creates
 *     the multicast object (lomo_mc_create; world > 1 also exports a POSIX
 *     file descriptor), the other ranks import it from rank 0's (pid, fd)
 *     (lomo_mc_import, pidfd_getfd), every rank adds its device
 *     (lomo_mc_add_device), and after ALL ranks have added theirs
 *     (a host barrier), binds local memory and maps both views
 *     (lomo_mc_bind: uc = this GPU's copy, mc = the multicast address).
 *     `obj` is an opaque handle; lomo_mc_free releases everything.
 *
 * Device barrier: every rank calls it with the same (channel, epoch) sequence,
 * epochs strictly increasing per channel (the caller counts).  It is one
 * stream-ordered kernel: a system-scope release of everything this stream
 * wrote before it, a signal to every peer, and an acquire-wait for every
 * peer's signal.  A wait longer than timeout_ns sets *err_dev = 2 and returns
 * (never hangs the GPU).  Pass &state->error: the step's status read then
 * surfaces the timeout.
 *   lomo_peer_barrier: sig_dev = DEVICE array of the world ranks' signal
 *     areas (each LOMO_PEER_SIGNAL_BYTES, IPC-mapped; sig_dev[rank] is own).
 *   lomo_mc_barrier: sig_mc / sig_uc = a LOMO_PEER_SIGNAL_BYTES area at the
 *     multicast / this rank's unicast address of a bound multicast object. */
#define LOMO_PEER_MAX 16
#define LOMO_PEER_CHANNELS 16
#define LOMO_PEER_SIGNAL_BYTES (8 * LOMO_PEER_CHANNELS * LOMO_PEER_MAX)
#define LOMO_E_UNSUPPORTED (-3) /* capability absent (e.g. no multicast) */
size_t lomo_ipc_handle_bytes(void);
int lomo_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out);
int lomo_ipc_open(const void* handle, void** dev_ptr);
int lomo_ipc_close(void* dev_ptr);
int lomo_ipc_free(void* dev_ptr);
int lomo_peer_barrier(void* const* sig_dev, int world, int rank, int channel, uint64_t epoch,
                      int64_t timeout_ns, int* err_dev, void* stream);
int lomo_mc_supported(int device);
int lomo_mc_create(int world, size_t bytes, uint64_t* obj, size_t* granted_bytes, int* fd);
int lomo_mc_import(int pid, int fd, size_t bytes, uint64_t* obj);
int lomo_mc_add_device(uint64_t obj, int device);
int lomo_mc_bind(uint64_t obj, int device, void** uc_ptr, void** mc_ptr);
int lomo_mc_free(uint64_t obj);
int lomo_mc_barrier(void* sig_mc, const void* sig_uc, int world, int channel, uint64_t epoch,
                    int64_t timeout_ns, int* err_dev, void* stream);
/* The same barriers with the epoch kept on the device: `epochs_dev` holds one
 * uint64 counter per channel (zero-initialised, this rank's own memory); the
 * barrier uses counter+1 and stores it back.  Every rank issues the same
 * sequence, so the counters agree -- and a CUDA graph that captured the
 * barrier advances them on every replay (GraphedShardedStep with K4). */
int lomo_peer_barrier_dev(void* const* sig_dev, uint64_t* epochs_dev, int world, int rank,
                          int channel, int64_t timeout_ns, int* err_dev, void* stream);
int lomo_mc_barrier_dev(void* sig_mc, const void* sig_uc, uint64_t* epochs_dev, int world,
                        int channel, int64_t timeout_ns, int* err_dev, void* stream);

/* ---- row-sparse embedding gradient (K1 on the rows a batch touched) ---- */
/* The reference's embedding VJP scatters dy into a dense [V, h] gradient;
 * LOMO's update leaves untouched rows unchanged (p - lr*0 == p), so the
 * gradient can live as one aggregated row per distinct id:
 * lomo_rows_aggregate: sorted_ids / perm = a stable sort of the ntok token
 * ids and the source positions; writes rows [ntok, h] (dtype) and row_ids
 * [ntok] -- run heads get the fp32 sum of their dy rows in token order
 * (rounded to dtype) and their id, other positions a zero row and -1.  K2 on
 * `rows` then equals K2 on the dense gradient up to summation order.
 * lomo_fused_update_rows: K1's arithmetic on p[row_ids[j], :] with
 * rows[j, :], skipping row_ids < 0; weight_decay must be 0 (LOMO_E_ARG:
 * decay changes every row). */
int lomo_rows_aggregate(const int64_t* sorted_ids, const int64_t* perm, const void* dy,
                        int64_t ntok, int64_t h, int dtype, void* rows, int64_t* row_ids,
                        void* stream);
int lomo_fused_update_rows(void* p, const void* rows, const int64_t* row_ids, int64_t nrows,
                           int64_t h, int dtype, int math, double lr, double clip_value,
                           double weight_decay, unsigned flags, const void* state,
                           void* stream);

/* ---- K5: weight-gradient GEMM with the update as its epilogue ---------- */
/* For a linear layer y = x W^T (W [out, in] row-major, x [tokens, in],
 * dy [tokens, out], all row-major, 16-bit): computes on the tensor cores
 *     p <- alpha * (dy^T x) + beta * p          (p == W, in place)
 * i.e. the LOMO update with alpha = -lr * coef / scale, beta = 1 - lr*wd, from
 * the fp32 accumulator -- the gradient dW is never written to memory.
 * Replaces the K1 launch of pass 2 under replay (replay.py); value clipping
 * is not linear in dW and stays on K1.  workspace: >= lomo_gemm_update_workspace
 * bytes of device memory (may be NULL when that is 0).  dtype: F16 or BF16;
 * out_features and in_features must be multiples of 8. */
int lomo_gemm_update(void* p, const void* dy, const void* x, int64_t out_features,
                     int64_t in_features, int64_t tokens, int dtype, double alpha,
                     double beta, void* workspace, size_t workspace_bytes, void* stream);
size_t lomo_gemm_update_workspace(int64_t out_features, int64_t in_features,
                                  int64_t tokens, int dtype);
/* As lomo_gemm_update, with alpha = coefs_dev[0] and beta = coefs_dev[1] read
 * from device memory at run time (graph-capturable); lomo_update_coefs
 * computes them on device from the step state:
 *   alpha = skip ? 0 : -state->lr * [coef] * [inv_scale],  beta = skip ? 1 : 1 - lr*wd
 * ([x] present when flags has LOMO_USE_COEF / LOMO_USE_SCALE). */
int lomo_gemm_update_dev(void* p, const void* dy, const void* x, int64_t out_features,
                         int64_t in_features, int64_t tokens, int dtype,
                         const float* coefs_dev, void* workspace, size_t workspace_bytes,
                         void* stream);
int lomo_update_coefs(const void* state, double weight_decay, unsigned flags,
                      float* coefs_dev, void* stream);

/* ---- K6: weight-gradient GEMM with the pass-1 probe as its epilogue ---- */
/* Replaces, for a linear layer, the weight-gradient GEMM dW = dy^T x followed
 * by a K2 launch over dW (stabilize.py:190-200 probe_hook): the tensor cores
 * compute dW tile by tile (the same mainloop as K5, so pass 2 sees
 * bit-identical accumulators) and the epilogue rounds each element to the
 * storage dtype, raises state->overflow if it is non-finite and accumulates
 * (g * inv_scale)^2 into norm slot `slot`, so the gradient is never read back.
 * grad_out receives the epilogue's store of dW: with LOMO_PROBE_KEEP_GRAD
 * the gradient itself ([out, in], dtype -- a retained gradient); otherwise no
 * gradient leaves the SM: grad_out is a 16-byte scratch (32 fp4 elements)
 * the epilogue's clipped store may touch, reusable at once (stream-ordered).
 * Without KEEP_GRAD in_features must be a multiple of 32.
 * flags: LOMO_USE_SCALE (LOMO_ACCUM_F64 is refused with LOMO_E_ARG: the
 * exactness mode keeps GEMM + K2).  workspace: >= lomo_gemm_probe_workspace
 * bytes of device memory, reused by every call on one stream.  Shapes as
 * lomo_gemm_update. */
int lomo_gemm_probe(const void* dy, const void* x, void* grad_out, int64_t out_features,
                    int64_t in_features, int64_t tokens, int dtype, int slot, unsigned flags,
                    void* state, void* workspace, size_t workspace_bytes, void* stream);
size_t lomo_gemm_probe_workspace(int64_t out_features, int64_t in_features, int64_t tokens,
                                 int dtype);
/* K6's second stage (also usable on its own): sum a [rows, ld] fp32 matrix of
 * partial sums of squares (first `cols` entries of each row valid; K6 passes
 * one row per 256-column tile of dW) in fixed order into norm slot `slot`
 * (one K2-style partial per row, finished by K3a); a NaN partial raises
 * state->overflow.  rows <= LOMO_PROBE_BLOCKS_PER_SLOT. */
int lomo_probe_rows(const float* partials_dev, int64_t rows, int64_t ld, int64_t cols, int slot,
                    void* state, void* stream);
/* lomo_probe_rows for `count` matrices in ceil(count/64) launches (host arrays). */
int lomo_probe_rows_multi(const float* const* partials_dev, const int64_t* rows,
                          const int64_t* ld, const int64_t* cols, const int* slots, int count,
                          void* state, void* stream);
/* Deferred K6 (flags & LOMO_DEFER_ROWS): each such call must get its own
 * workspace; after the batch, this reduces every call's partial sums into its
 * slot (one launch per 64 calls instead of one per call).  Host arrays. */
int lomo_gemm_probe_finish(void* const* workspaces, const int64_t* out_features,
                           const int64_t* in_features, const int* slots, int count, int dtype,
                           void* state, void* stream);

/* Number of SMs the library sized its grids for (device of the current
 * context); 0 if no device. */
int lomo_num_sms(void);

#ifdef __cplusplus
}
#endif

#endif /* LOMO_B200_H */
