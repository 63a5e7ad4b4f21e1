/*
 * dsp_b200.h -- C ABI of the B200-native Diversely-Stale-Parameters (DSP)
 * train step (arXiv 1909.02625).  Plain pointers and sizes only; no torch
 * types.  Every function returns 0 on success or a DSP_E* code; the message
 * of the last failure on the calling thread is in dsp_last_error().
 *
 * The reference (`stalepipe`, pure Python/numpy) has no FFI; its per-block
 * work is three Python calls inside TrainEngine._iterate_block
 * (/root/reference/pkg/src/stalepipe/pipeline.py:538-606):
 *
 *   block_forward(block, h_in, record)   blocks.py:96-118   -> dsp_block_forward
 *   softmax_xent(logits, labels)         tensor.py:86-111   -> dsp_block_loss
 *   block_backward(block, tape, u)       blocks.py:121-154  -> dsp_block_backward
 *   g = grad + wd*params; apply_update   pipeline.py:591-596,
 *                                        optim.py:48-109    -> dsp_block_update
 *
 * The queues / FIFO indexing (pipeline.py:148-205, 483-513) stay on the host
 * side (Python mirror of the reference) and pass device ring-slot pointers in.
 * INTEGRATION.md shows the ctypes binding a `stalepipe` maintainer would add.
 */
#ifndef DSP_B200_H_
#define DSP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ error codes */
#define DSP_OK 0
#define DSP_E_INVALID 1   /* bad argument / shape (reference: ShapeError, ValueError) */
#define DSP_E_CUDA 2      /* CUDA runtime failure */
#define DSP_E_STATE 3     /* call order violated (reference: RuntimeError "tape already consumed") */
#define DSP_E_NONFINITE 4 /* non-finite values (reference: NonFiniteError, tensor.py:23-37) */

/* ------------------------------------------------------------ enums */
#define DSP_DTYPE_BF16 0 /* bf16 storage, kind::f16 tensor-core MMA, fp32 accumulate */
#define DSP_DTYPE_F32 1  /* fp32 storage, 3xTF32 on kind::tf32 tensor cores (fp32-faithful), fp32 accumulate */

#define DSP_IGEMM_FPROP 0
#define DSP_IGEMM_DGRAD 1
#define DSP_IGEMM_WGRAD 2

/* Layer kinds.  0..2 are the reference's own (blocks.py:21-33); the rest are
 * the CNN kinds the BASELINE configs need (ResNet units at residual-unit
 * granularity). */
#define DSP_LAYER_DENSE 0
#define DSP_LAYER_RELU 1
#define DSP_LAYER_TANH 2
#define DSP_LAYER_CONV_BN_RELU 10 /* conv kxk + BatchNorm + ReLU (stem) */
#define DSP_LAYER_BASIC_UNIT 11   /* 2x conv3x3-BN (+1x1 projection-BN) + residual + ReLU */
#define DSP_LAYER_BOTTLENECK 12   /* conv1x1-BN-ReLU, conv3x3-BN-ReLU, conv1x1-BN, shortcut, ReLU */
#define DSP_LAYER_AVGPOOL 13      /* global average pool (B,H,W,C) -> (B,C) */
#define DSP_LAYER_MAXPOOL 14      /* 3x3 stride-2 pad-1 max pool (ResNet-50 stem) */

#define DSP_RULE_SGD 0
#define DSP_RULE_SUM 1
/* Bias-corrected Adam: an EXTENSION for BASELINE configs[2] (the reference rejects rule "adam",
 * optim.py:70-71; parity is against this repo's restatement oracle/dsp_ref.py adam_step only). */
#define DSP_RULE_ADAM 2
/* fp32 Adam state of an n-parameter block: m[n], v[n], then an int64 step counter at float
 * offset 2n (counts applied updates; zero = fresh, OptimizerState.for_params). */
#define DSP_ADAM_STATE_BYTES(n) ((size_t)(n) * 8 + 8)

/* ------------------------------------------------------------ kernel level */
typedef struct {
  int32_t nimg;            /* batch */
  int32_t H, W, C;         /* input spatial size, channels (padded to a multiple of 8) */
  int32_t P, Q, K;         /* output spatial size, channels (padded to a multiple of 8) */
  int32_t R, S, stride, pad;
} dsp_conv_geom_t;

/* One BatchNorm whose backward statistics a DGRAD epilogue accumulates (see
 * dsp_igemm_args_t.bnb): the BN sits below the conv whose input gradient the
 * DGRAD produces, g = dX * (mask > 0) is its upstream gradient. */
typedef struct {
  const void* y;           /* the BN's input (conv output), storage dtype, same [M][ldd] layout as D */
  const float* stat;       /* its forward statistics block: row 0 mean, row 1 invstd ([4][N]) */
  const float* gamma;      /* [c_real] */
  float* dgamma;           /* out [c_real]: sum g * xhat */
  float* dbeta;            /* out [c_real]: sum g */
  float* coef;             /* out [3][N]: gamma*invstd, mean(g), mean(g*xhat) (0 past c_real) */
} dsp_bnb_target_t;

typedef struct {
  dsp_conv_geom_t geom;
  int32_t M, N, Kd;        /* GEMM extents (see igemm.cu header comment) */
  const void* A;           /* FPROP/WGRAD: X (NHWC); DGRAD: dY (NHWC) */
  const void* B;           /* FPROP/DGRAD: packed weights [K][R][S][C]; WGRAD: dY */
  void* D;                 /* FPROP/DGRAD: output [M][ldd]; WGRAD: fp32 partials [splits][M][N] */
  int32_t ldd;
  int32_t out_f32;         /* FPROP/DGRAD: 1 = store fp32 instead of the storage dtype (0 or 1; other values are
                              rejected -- builds with -DIG_TRACE_BUILD read diagnostic switches from the
                              upper bits) */
  const void* residual;    /* optional [M][ldd] added in the epilogue */
  const float* bias;       /* optional [N] added in the epilogue */
  float* stats;            /* optional BatchNorm partials, one row per CTA: [DSP_IGEMM_MAX_CTAS][2][N]
                              (sum, sum of squares of the stored values) */
  int32_t kb_per_split;    /* WGRAD split-K: K blocks per split */
  int32_t n_valid;         /* FPROP/DGRAD: columns >= n_valid are stored as 0 (0 = all N valid) */
  /* FPROP fused BatchNorm finalize (optional, needs stats): per n-tile of the
   * launch, the last CTA owning it reduces that tile's per-CTA partials in fixed
   * order and writes stat_out[4][N] = mean, invstd, gamma*invstd,
   * beta - mean*gamma*invstd for its columns (columns >= n_valid get zeros). Large grids
   * finalize in two levels (groups of 16 CTAs, then the group sums).
   * sem: DSP_IGEMM_SEM_INTS device ints, 0 on entry (the kernel leaves them 0 again). */
  float* stat_out;
  const float* gamma;
  const float* beta;
  int32_t* sem;
  int64_t* trace;          /* optional profiling (builds with -DIG_TRACE_BUILD only): clock64() stamps of CTA 0's
                              pipeline events (slots 0..191), then per-CTA %globaltimer stamps (8 slots per CTA) */
  /* DGRAD fused BatchNorm-backward statistics (optional; needs stats and sem):
   * with g = stored dX * (bnb_mask > 0), per column the kernel accumulates sum g
   * and sum g * xhat_t for each of bnb_count (1 or 2) BNs sharing g (stats rows:
   * [CTA][1 + bnb_count][N]); the last CTA finalizes into bnb[t].dgamma / dbeta /
   * coef, exactly what bn_bwd_stats writes, for channels < bnb_c_real. bnb_mask = NULL (one target
   * only): the BN's output is relu(y*scale + shift) with no residual, so the mask is recomputed from
   * bnb[0].y and its stat rows 2-3 (scale, shift) instead of read. */
  const void* bnb_mask;
  int32_t bnb_count;
  int32_t bnb_c_real;
  dsp_bnb_target_t bnb[2];
  /* DGRAD (optional): the weights transposed per tap, [Cin_p][R][S][Cout_p] bf16 -- lets
   * stride-1 DGRAD load K-major weight boxes with TMA and use halo tiles like FPROP. */
  const void* B_t;
  /* DGRAD bnb (optional, bf16, takes precedence over bnb_mask): the mask as bits, one byte per 8
   * columns of every row ([M][ldd / 8]), bit i = column 8j + i of the BN's output > 0 (what the
   * forward's BN-apply wrote beside the output). */
  const uint8_t* bnb_mask_bits;
} dsp_igemm_args_t;

#define DSP_IGEMM_MAX_CTAS 444
#define DSP_IGEMM_SEM_INTS 1024 /* ticket ints a fused-finalize launch may use (dsp_igemm_args_t.sem) */

/* Implicit-GEMM conv/dense on tcgen05 tensor cores (igemm.cu).  `splits` is the
 * WGRAD split-K factor (ignored otherwise). */
int dsp_igemm(int mode, int dtype, const dsp_igemm_args_t* args, int splits, void* stream);

/* Per-block parameter update (optim.py:48-109 + pipeline.py:591-596), flat
 * vectors of length n.  The fp64 variant reproduces the reference's IEEE op
 * order bit for bit (no FMA contraction); the fp32 variant is the engine's.
 *   g      = grad + wd*x        (only if wd != 0)
 *   SGD:   x' = x - lr*g
 *   SUM:   y = x - lr*g; ys' = x - slr*g; x' = beta==0 ? y : y + beta*(ys' - ys)
 * slr = s*lr is formed by the caller (optim.py:92 evaluates (state.s*lr)).
 * grad_sq (optional, device) receives sum(grad^2) (pre-WD, pipeline.py:602).
 * ys may be NULL for SGD; y (optional) receives y for API fidelity (optim.py:97). */
int dsp_update_f64(int rule, int64_t n, double* x, const double* grad, double* ys, double* y, double lr,
                   double slr, double beta, double wd, double* grad_sq, void* stream);
int dsp_update_f32(int rule, int64_t n, float* x, const float* grad, float* ys, double lr, double slr,
                   double beta, double wd, float* grad_sq, void* stream);

/* ------------------------------------------------------------ block level */
typedef struct {
  int32_t kind;            /* DSP_LAYER_* */
  int32_t in_c, in_h, in_w;   /* real (unpadded) input shape; dense: (in_dim, 1, 1) */
  int32_t out_c, out_h, out_w;
  int32_t mid_c;           /* bottleneck width */
  int32_t stride;
  int32_t ksize;           /* CONV_BN_RELU kernel size */
  int32_t bias;            /* DENSE: has bias */
  int32_t reserved;
  int64_t param_offset;    /* into the block's flat fp32 parameter vector */
  int64_t param_count;
} dsp_layer_desc_t;

typedef struct dsp_block dsp_block_t;

/* Plan a block: a consecutive run of layers (blocks.py:65-93, 229-252).
 * is_last: the block ends in logits and owns the loss (pipeline.py:575-576). */
int dsp_block_create(const dsp_layer_desc_t* layers, int n_layers, int batch, int dtype, int is_last,
                     dsp_block_t** out);
void dsp_block_destroy(dsp_block_t* blk);
/* Device bytes the caller must provide to dsp_block_bind (activations, tape,
 * BN statistics, packed weights, split-K scratch). */
int64_t dsp_block_workspace_bytes(const dsp_block_t* blk);
/* Element counts (whole batch, padded NHWC) of the block input / output activation. */
int64_t dsp_block_in_elems(const dsp_block_t* blk);
int64_t dsp_block_out_elems(const dsp_block_t* blk);
int64_t dsp_block_param_count(const dsp_block_t* blk);
/* Bind device memory: workspace, flat fp32 params and grads (param_count each). */
int dsp_block_bind(dsp_block_t* blk, void* workspace, float* params, float* grads, void* stream);
/* Re-pack the storage-dtype weight shadow from the fp32 params (after an external write). */
int dsp_block_pack(dsp_block_t* blk, void* stream);
/* Make `twin` (planned from the same layer program and batch, bound to its own workspace and
 * to the primary's params) a FORWARD TWIN of `primary`: its convs read the primary's packed
 * weight shadow, and dsp_block_pack on it becomes a no-op.  A block's fresh forward
 * (pipeline.py:564) then runs on the twin, on its own stream, concurrently with the primary's
 * recompute + backward (pipeline.py:566-582); the caller joins it before the update.  Call
 * again after re-binding the primary. */
int dsp_block_share_weights(dsp_block_t* twin, const dsp_block_t* primary);

/* block_forward: x (padded input, storage dtype) -> y (padded output).
 * record=1 keeps the tape for dsp_block_backward (recompute pass); y may be
 * NULL when record=1 (the reference discards it, pipeline.py:566). For the
 * last block the output is fp32 logits [B][classes padded to 8] kept in the
 * workspace; if y is non-NULL they are also copied there. */
int dsp_block_forward(dsp_block_t* blk, const void* x, void* y, int record, void* stream);
/* softmax_xent on the recorded logits (last block only): writes the mean loss
 * to *loss_dev (device fp32) and keeps dlogits as the backward upstream. */
int dsp_block_loss(dsp_block_t* blk, const int64_t* labels_dev, float* loss_dev, void* stream);
/* Bias-corrected Adam (DSP_RULE_ADAM extension), flat vectors of length n:
 *   g = grad + wd*x (only if wd != 0); m' = b1*m + (1-b1)*g; v' = b2*v + (1-b2)*g*g
 *   x' = x - (lr*(m'/bc1)) / (sqrt(v'/bc2) + eps),  bc_i = 1 - b_i^t
 * t = *tstep + 1 when tstep (device int64) is given -- the call then also increments it --,
 * else bc1/bc2 are taken from the host.  The fp64 variant keeps the restatement's IEEE op
 * order (no FMA contraction). */
int dsp_update_adam_f64(int64_t n, double* x, const double* grad, double* m, double* v, int64_t* tstep, double bc1,
                        double bc2, double lr, double b1, double b2, double eps, double wd, double* grad_sq,
                        void* stream);
int dsp_update_adam_f32(int64_t n, float* x, const float* grad, float* m, float* v, int64_t* tstep, double bc1,
                        double bc2, double lr, double b1, double b2, double eps, double wd, float* grad_sq,
                        void* stream);

/* block_backward on the recorded tape.  upstream: padded dY (NULL for the
 * last block, which uses dlogits).  grad_in: padded dX or NULL to skip the
 * input gradient (block 0).  Writes the flat fp32 parameter gradient. */
int dsp_block_backward(dsp_block_t* blk, const void* upstream, void* grad_in, void* stream);
/* Update the bound params from the bound grads and re-pack the weight shadow, in ONE launch (a
 * tile table covers the parameter vector: each weight tile is updated, written to the storage-
 * dtype shadow and, through shared memory, to its transposed DGRAD copy; the grad-norm partials
 * are summed by the last CTA into *grad_sq_out). apply = 0: grad norm only (a discarded warmup
 * update, pipeline.py:594). A non-finite gradient (after weight decay) in an applied update sets
 * the block's sticky non-finite flag (dsp_block_nonfinite). */
int dsp_block_update(dsp_block_t* blk, int rule, float* ys, double lr, double slr, double beta, double wd,
                     int apply, float* grad_sq_out, void* stream);

/* Sticky non-finite flags of a block -- the device side of the reference's NonFiniteError
 * (tensor.py:34-37 / 101-111, optim.py:53 / 89), checked at sync points instead of raising in the
 * middle of an asynchronous step: bit 0 = dsp_block_loss produced a non-finite loss, bit 1 = an
 * applied dsp_block_update met a non-finite gradient. One 4-byte device->host copy on `stream` and
 * a stream synchronize; clear != 0 resets the flags. */
#define DSP_NONFINITE_LOSS 1
#define DSP_NONFINITE_GRAD 2
int dsp_block_nonfinite(dsp_block_t* blk, int clear, int* flags_out, void* stream);

/* Adam variant of dsp_block_update: state = DSP_ADAM_STATE_BYTES(param_count) bytes of device
 * memory laid out as described at DSP_ADAM_STATE_BYTES (the step counter advances on apply). */
int dsp_block_update_adam(dsp_block_t* blk, void* state, double lr, double b1, double b2, double eps, double wd,
                          int apply, float* grad_sq_out, void* stream);

/* ------------------------------------------------------------ utilities */
/* Host fp64 batch -> padded device activation (storage dtype).  x_dev points
 * to a device copy of the fp32 batch [B][C*H*W] in the reference's flattened
 * (C,H,W) order (CNN) or [B][D] (dense). */
int dsp_pack_input(const float* x_dev, void* out, int batch, int c, int h, int w, int c_pad, int dtype,
                   int nchw, void* stream);
int dsp_unpack_output(const void* in, float* out_dev, int batch, int c, int h, int w, int c_pad, int dtype,
                      int nchw, void* stream);
/* Batch batch_no of the synthetic pool synthetic_batches(n, B, (c,h,w), num_classes, seed)
 * (x ~ SeededRng(seed).normal, labels = floor(SeededRng(derive_seed(seed,1))
 * .uniform * C), rng.py:47-88) generated on the device: act_out = packed NHWC activation
 * (dtype, channels padded to c_pad), labels_out = int64 [B]; either may be NULL. */
int dsp_synth_batch(uint64_t seed, int64_t batch_no, int batch, int c, int h, int w, int c_pad, int num_classes,
                    int dtype, void* act_out, int64_t* labels_out, void* stream);
/* Straggler injection: a one-thread kernel that keeps the stream busy
 * for ns nanoseconds (the device counterpart of the reference's RuntimeStraggler sleeps). */
int dsp_device_sleep(int64_t ns, void* stream);
const char* dsp_last_error(void);
int dsp_abi_version(void);
/* Number of kernels this library has launched in the process (bench evidence). */
int64_t dsp_launch_count(void);

/* ------------------------------------------------------------ engine level
 * The whole DSP train step behind one handle: the reference's
 * TrainEngine(model, config, data, schedule, rule, beta, s, weight_decay) +
 * run(n) + log (pipeline.py:451-606, 610-660, 664): all K blocks on one device,
 * or one device per block (dsp_config_t.multi_device). The queue config is validated by the caller exactly as
 * validate_config does (pipeline.py:85-128); dsp_create re-checks Eq.(5) and
 * returns DSP_E_INVALID naming the first violated constraint. */
#define DSP_MAX_BLOCKS 8
#define DSP_WARMUP_FAITHFUL 0 /* "faithful_zero_updates" */
#define DSP_WARMUP_DISCARD 1  /* "discard_warmup_updates" */

typedef struct {
  int32_t K;                      /* blocks, 1..DSP_MAX_BLOCKS */
  int32_t p[DSP_MAX_BLOCKS];      /* forward queue delays (p[K-1] = 0) */
  int32_t m[DSP_MAX_BLOCKS];      /* staleness per block (m[K-1] >= 0) */
  int32_t warmup;                 /* DSP_WARMUP_* */
  int32_t batch;                  /* B */
  int32_t dtype;                  /* DSP_DTYPE_BF16 (bf16 storage) or DSP_DTYPE_F32 (fp32 storage, 3xTF32) */
  int32_t in_c, in_h, in_w;       /* one sample of the host batches, (C,H,W) flattened C-major */
  int32_t num_classes;            /* labels must lie in [0, num_classes) */
  int32_t n_layers[DSP_MAX_BLOCKS];
  const dsp_layer_desc_t* layers; /* all blocks' layers back to back; param_offset relative to its block */
  int32_t use_graphs;             /* replay each step as a CUDA graph once the zero prefill has drained */
  int32_t device;                 /* CUDA device ordinal (all blocks, unless multi_device) */
  /* multi_device = 1: block k runs on device_of_block[k] (one GPU per block is the
   * reference's one worker per block, pipeline.py:622-660). Rings live on the consumer's device and
   * the producer's last kernel stores each packet into the peer slot over NVLink (peer access is
   * enabled along every cross-device FIFO edge); each device replays its own step graph, ordered
   * after its neighbours' previous step by events. */
  int32_t multi_device;
  int32_t device_of_block[DSP_MAX_BLOCKS];
} dsp_config_t;

typedef struct {
  int64_t step;         /* block step n */
  int32_t block;
  int32_t has_loss;     /* last block only */
  int64_t batch_index;  /* stale tag n - cum_p[k] - m_k (negative: zero prefill packet) */
  double loss;          /* mean cross-entropy of the stale batch (NaN unless has_loss) */
  double grad_norm;     /* ||grad||_2 before weight decay (pipeline.py:602) */
} dsp_log_record_t;

typedef struct dsp_engine dsp_engine_t;

int dsp_create(const dsp_config_t* cfg, dsp_engine_t** out);
/* Parameters of block k: n = param_count values, host float64 (on_device = 0,
 * the reference's dtype) or device fp32 (on_device = 1). Resets the optimizer
 * state of the block (ys_0 = x_0, optim.py:82). */
int dsp_set_params(dsp_engine_t* eng, int k, const void* src, size_t n, int on_device);
int dsp_get_params(dsp_engine_t* eng, int k, double* dst, size_t n);
size_t dsp_param_count(dsp_engine_t* eng, int k);
/* rule: DSP_RULE_SGD / DSP_RULE_SUM; lr(n) = base_lr * prod(factors[i] for decay_steps[i] <= n)
 * (optim.py:38-45); wd couples into the gradient (pipeline.py:591-593). */
int dsp_set_optimizer(dsp_engine_t* eng, int rule, double beta, double s, double wd, double base_lr,
                      const int64_t* decay_steps, const double* factors, int n_decay);
/* Adam hyper-parameters (rule DSP_RULE_ADAM; defaults 0.9 / 0.999 / 1e-8, oracle adam_step).
 * beta / s of dsp_set_optimizer are unused by Adam. */
int dsp_set_adam(dsp_engine_t* eng, double beta1, double beta2, double eps);
/* n_steps DSP steps. x: host float32 [n_steps][B][C*H*W], labels: host int64
 * [n_steps][B] -- batch n of this call is the data stream's next batch. Each
 * step copies its batch host->device and its loss / grad-norm row device->host
 * (pinned, asynchronous); returns after the last step completed, with
 * DSP_E_NONFINITE if any block's non-finite flag is set (dsp_block_nonfinite;
 * the reference's NonFiniteError). */
int dsp_run(dsp_engine_t* eng, int n_steps, const float* x, const int64_t* labels);
/* Records of all steps so far, sorted by (step, block); *n = how many (<= cap written). */
int dsp_read_log(dsp_engine_t* eng, dsp_log_record_t* recs, size_t cap, size_t* n);
int64_t dsp_steps_done(dsp_engine_t* eng);
void dsp_destroy(dsp_engine_t* eng);

/* Live kernel timing (bench.py roofline): while armed, every dsp_igemm-class launch with
 * (mode, N, M) records events[2i] before and events[2i+1] after it on its own stream (also
 * inside CUDA-graph capture), i = 0, 1, ... up to n_pairs; dsp_probe_reset() restarts at 0 and
 * returns how many launches were probed. events: cudaEvent_t handles; NULL disarms. mode: a
 * DSP_IGEMM_* value in bits 0-7; bits 8+ (if nonzero) also require the launch's Kd to equal them. */
int dsp_probe_arm(int mode, int n, int64_t m, void* const* events, int n_pairs);
int dsp_probe_reset(void);

/* Step-graph execution (the engine's replacement for the reference's per-step
 * Python loop, pipeline.py:416-449).  graph: a captured cudaGraph_t; flags:
 * DSP_GRAPH_NODE_PRIORITY honours each kernel node's priority (inherited from the
 * capturing stream), so the pipeline's critical-path block is scheduled first. */
#define DSP_GRAPH_NODE_PRIORITY 1
int dsp_graph_instantiate(void* graph, int flags, void** exec_out);
int dsp_graph_launch(void* exec, void* stream);
int dsp_graph_destroy(void* exec);

#ifdef __cplusplus
}
#endif
#endif /* DSP_B200_H_ */
