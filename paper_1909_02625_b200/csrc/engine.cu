// The DSP train step behind one C handle (include/dsp_b200.h, "engine level").
//
// Native counterpart of the reference's TrainEngine (/root/reference/pkg/src/stalepipe/
// pipeline.py:451-606 construction + _iterate_block, 610-660 run, 664 log) for K blocks on one
// GPU or -- with dsp_config_t.multi_device -- block k on device_of_block[k] (the reference's
// one-worker-per-block, pipeline.py:622-660, as one GPU per block), built on the block executor
// (block.cu). The FIFOs are not materialised as queues: every packet lives in a device ring slot
// chosen by the closed forms of SURVEY.md Appendix A --
//   block k at step n: fresh tag n - cum_p[k], stale tag n - cum_p[k] - m_k;
//   its fresh input is block k-1's output of step n - p_{k-1}, its stale input
//   that of step n - m_k - p_{k-1}, its upstream gradient block k+1's input
//   gradient of step n - q_{k+1}; a negative step means a zero prefill packet
//   (pipeline.py:483-513, 524-528)
// -- so the batch-tag protocol check of pipeline.py:567-572 holds by construction.
// Rings live on the CONSUMER's device: a producer's last kernel (BN-apply of its forward, the
// DGRAD of its backward) stores its packet straight into the peer ring slot over NVLink (peer
// access), so the stage-to-stage transfer is fused into the producing kernel's epilogue and
// overlaps the rest of the producer's step. Step n of a device starts after step n-1 of every
// device holding a neighbour of one of its blocks (every packet read at step n was written at
// step <= n-1, every slot written at step n was last read at step <= n-1).
// Ring depth R exceeds every packet lifetime, so from the step on which no zero packet is read
// any more the device work of step n depends only on n mod R: each device captures its blocks'
// step once per phase into a CUDA graph (its blocks on forked streams) and replays it; a phase is
// re-captured when its learning rates / update flags change.
#include "abi_internal.h"
#include "common.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace {

using dsp::set_error;

struct Phase {
  cudaGraphExec_t exec = nullptr;
  std::vector<double> lr;   // signature: per-block lr and update flag
  std::vector<int> apply;
};

constexpr int kMaxDev = DSP_MAX_BLOCKS;  // distinct devices of one engine

}  // namespace

struct dsp_engine {
  dsp_config_t cfg{};
  int K = 0, B = 0, R = 0, D = 0;  // D = C*H*W of one input sample
  int cum_p[DSP_MAX_BLOCKS + 1] = {};
  int q[DSP_MAX_BLOCKS] = {};
  int horizon = 0;
  std::vector<dsp_layer_desc_t> layers;
  // devices: ndev distinct ordinals devs[j]; block k runs on devs[dj[k]]
  int ndev = 1;
  int devs[kMaxDev] = {};
  int dj[DSP_MAX_BLOCKS] = {};
  bool nbr[kMaxDev][kMaxDev] = {};  // device j waits for device i's previous step
  dsp_block_t* blk[DSP_MAX_BLOCKS] = {};
  // forward twins (k < K-1): the fresh forward runs on twin[k] / fstream[k], beside the
  // recompute + backward of blk[k] on the block stream, joined before the update
  dsp_block_t* twin[DSP_MAX_BLOCKS] = {};
  void* tws[DSP_MAX_BLOCKS] = {};
  cudaStream_t fstream[DSP_MAX_BLOCKS] = {};
  cudaEvent_t fev_fork[DSP_MAX_BLOCKS] = {}, fev_join[DSP_MAX_BLOCKS] = {};
  int64_t nparam[DSP_MAX_BLOCKS] = {};
  int64_t in_elems[DSP_MAX_BLOCKS] = {}, out_elems[DSP_MAX_BLOCKS] = {};
  void* ws[DSP_MAX_BLOCKS] = {};
  float* params[DSP_MAX_BLOCKS] = {};
  float* grads[DSP_MAX_BLOCKS] = {};
  float* ys[DSP_MAX_BLOCKS] = {};
  // rings (slot = step mod R), each on its consumer's device
  std::vector<void*> ring_out[DSP_MAX_BLOCKS], ring_gin[DSP_MAX_BLOCKS];
  std::vector<void*> ring_in;        // block 0's device
  std::vector<int64_t*> ring_lab;    // the last block's device
  void* zero_act[kMaxDev] = {};      // read-only zero packet (largest activation) per device
  int64_t* zero_lab = nullptr;       // the last block's device
  // input staging, double-buffered: batch n goes pinned host -> xdev[n&1] -> ring slot on the
  // copy stream of block 0's device (labels: of the last block's device), overlapping step n-1
  float* xdev[2] = {};
  float* pin_x[2] = {};
  int64_t* pin_l[2] = {};
  cudaEvent_t pin_ev[2] = {};   // copy of batch n done (pinned slot and xdev[n&1] free again)
  cudaEvent_t lab_ev[2] = {};
  cudaStream_t copy_stream = nullptr, lab_stream = nullptr;
  float* slots[kMaxDev] = {};    // [R][K][2] loss, grad_sq of the step in that phase (device j's blocks)
  std::vector<float*> host_log[kMaxDev];  // pinned chunks of LOG_CHUNK rows x K x 2, per device
  static constexpr int LOG_CHUNK = 4096;
  // optimizer
  int rule = DSP_RULE_SGD;
  double beta = 0.0, s = 1.0, wd = 0.0, base_lr = 0.01;
  double adam_b1 = 0.9, adam_b2 = 0.999, adam_eps = 1e-8;  // rule DSP_RULE_ADAM (extension)
  std::vector<std::pair<int64_t, double>> decays;
  // execution: per device a step stream (graphs launch here) and its per-step done events
  cudaStream_t dstream[kMaxDev] = {};
  cudaEvent_t done_ev[kMaxDev][2] = {};
  cudaEvent_t fork_ev[kMaxDev] = {};
  cudaStream_t bstream[DSP_MAX_BLOCKS] = {};
  cudaEvent_t join_ev[DSP_MAX_BLOCKS] = {};
  std::vector<Phase> phases[kMaxDev];
  int64_t steps = 0;  // steps done (all blocks advance together)
};

namespace {

int check(cudaError_t e, const char* what) { return dsp::cuda_check(e, what); }
#define ENG_CUDA(expr) DSP_TRY(check((expr), #expr))

int dev_of(const dsp_engine* e, int k) { return e->devs[e->dj[k]]; }

double lr_at(const dsp_engine* e, int64_t n) {
  double lr = e->base_lr;
  for (const auto& d : e->decays)
    if (n >= d.first) lr *= d.second;
  return lr;
}

int validate(const dsp_config_t& c) {
  const int K = c.K;
  if (K < 1 || K > DSP_MAX_BLOCKS) return set_error(DSP_E_INVALID, "dsp_create: K = %d outside [1, %d]", K, DSP_MAX_BLOCKS);
  if (c.p[K - 1] != 0)
    return set_error(DSP_E_INVALID, "ConfigError p_last_zero[%d]: p[%d] = %d must be 0", K - 1, K - 1, c.p[K - 1]);
  for (int k = 0; k < K - 1; ++k)
    if (c.p[k] <= 0) return set_error(DSP_E_INVALID, "ConfigError p_positive[%d]: p[%d] = %d must be > 0", k, k, c.p[k]);
  for (int k = 0; k < K - 1; ++k)
    if (c.m[k] <= 0) return set_error(DSP_E_INVALID, "ConfigError m_positive[%d]: m[%d] = %d must be > 0", k, k, c.m[k]);
  if (c.m[K - 1] < 0)
    return set_error(DSP_E_INVALID, "ConfigError m_last_nonneg[%d]: m[%d] = %d must be >= 0", K - 1, K - 1, c.m[K - 1]);
  for (int k = 1; k < K; ++k) {
    const int qk = c.m[k - 1] - c.p[k - 1] - c.m[k];
    if (qk <= 0)
      return set_error(DSP_E_INVALID, "ConfigError q_positive[%d]: q[%d] = m[%d]-p[%d]-m[%d] = %d-%d-%d = %d <= 0", k, k,
                       k - 1, k - 1, k, c.m[k - 1], c.p[k - 1], c.m[k], qk);
  }
  if (c.warmup != DSP_WARMUP_FAITHFUL && c.warmup != DSP_WARMUP_DISCARD)
    return set_error(DSP_E_INVALID, "dsp_create: unknown warmup policy %d", c.warmup);
  if (c.batch <= 0 || c.in_c <= 0 || c.in_h <= 0 || c.in_w <= 0 || c.num_classes <= 0 || !c.layers)
    return set_error(DSP_E_INVALID, "dsp_create: bad batch / input shape / classes / layers");
  if (c.dtype != DSP_DTYPE_BF16 && c.dtype != DSP_DTYPE_F32)
    return set_error(DSP_E_INVALID, "dsp_create: dtype %d is neither DSP_DTYPE_BF16 nor DSP_DTYPE_F32", c.dtype);
  for (int k = 0; k < K; ++k)
    if (c.n_layers[k] <= 0) return set_error(DSP_E_INVALID, "dsp_create: block %d has no layers", k);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
  for (int k = 0; k < K; ++k) {
    const int d = c.multi_device ? c.device_of_block[k] : c.device;
    if (d < 0 || d >= ndev) return set_error(DSP_E_INVALID, "dsp_create: block %d on device %d, %d device(s) visible", k, d, ndev);
  }
  return DSP_OK;
}

template <typename T>
int dmalloc(T** p, size_t bytes, bool zero = false) {
  ENG_CUDA(cudaMalloc((void**)p, std::max<size_t>(bytes, 16)));
  if (zero) ENG_CUDA(cudaMemset(*p, 0, std::max<size_t>(bytes, 16)));
  return DSP_OK;
}

// device pointer of the packet block k reads at step n (all on block k's device)
const void* fresh_in(const dsp_engine* e, int k, int64_t n) {
  if (k == 0) return e->ring_in[n % e->R];
  const int64_t src = n - e->cfg.p[k - 1];
  return src >= 0 ? e->ring_out[k - 1][src % e->R] : e->zero_act[e->dj[k]];
}
const void* stale_in(const dsp_engine* e, int k, int64_t n) {
  const int64_t f = n - e->cfg.m[k];  // the step this packet was fresh
  if (f < 0) return e->zero_act[e->dj[k]];
  return fresh_in(e, k, f);
}
const int64_t* stale_labels(const dsp_engine* e, int64_t n) {
  const int64_t tag = n - e->cum_p[e->K - 1] - e->cfg.m[e->K - 1];
  return tag >= 0 ? e->ring_lab[tag % e->R] : e->zero_lab;
}
const void* upstream(const dsp_engine* e, int k, int64_t n) {
  const int64_t src = n - e->q[k + 1];
  return src >= 0 ? e->ring_gin[k + 1][src % e->R] : e->zero_act[e->dj[k]];
}
bool apply_update(const dsp_engine* e, int k, int64_t n) {
  const int64_t stale_tag = n - e->cum_p[k] - e->cfg.m[k];
  return !(e->cfg.warmup == DSP_WARMUP_DISCARD && stale_tag < 0);
}

// Algorithm-2 body of block k at step n (pipeline.py:538-606) on stream st (block k's device).
int issue_block(dsp_engine* e, int k, int64_t n, cudaStream_t st) {
  const int K = e->K;
  const int ph = (int)(n % e->R);
  float* loss_slot = e->slots[e->dj[k]] + ((size_t)ph * K + k) * 2;
  if (k < K - 1) {
    if (e->twin[k]) {  // fresh forward on the twin's stream, overlapping recompute + backward
      ENG_CUDA(cudaEventRecord(e->fev_fork[k], st));
      ENG_CUDA(cudaStreamWaitEvent(e->fstream[k], e->fev_fork[k], 0));
      DSP_TRY(dsp_block_forward(e->twin[k], fresh_in(e, k, n), e->ring_out[k][ph], 0, e->fstream[k]));
      ENG_CUDA(cudaEventRecord(e->fev_join[k], e->fstream[k]));
    } else {
      DSP_TRY(dsp_block_forward(e->blk[k], fresh_in(e, k, n), e->ring_out[k][ph], 0, st));
    }
    DSP_TRY(dsp_block_forward(e->blk[k], stale_in(e, k, n), nullptr, 1, st));
    DSP_TRY(dsp_block_backward(e->blk[k], upstream(e, k, n), k > 0 ? e->ring_gin[k][ph] : nullptr, st));
    // the update rewrites the packed weights the fresh forward reads
    if (e->twin[k]) ENG_CUDA(cudaStreamWaitEvent(st, e->fev_join[k], 0));
  } else {
    DSP_TRY(dsp_block_forward(e->blk[k], stale_in(e, k, n), nullptr, 1, st));
    DSP_TRY(dsp_block_loss(e->blk[k], stale_labels(e, n), loss_slot, st));
    DSP_TRY(dsp_block_backward(e->blk[k], nullptr, k > 0 ? e->ring_gin[k][ph] : nullptr, st));
  }
  const double lr = lr_at(e, n);
  if (e->rule == DSP_RULE_ADAM)  // ys[k] holds the Adam state (m, v, step counter)
    return dsp_block_update_adam(e->blk[k], e->ys[k], lr, e->adam_b1, e->adam_b2, e->adam_eps, e->wd,
                                 apply_update(e, k, n) ? 1 : 0, loss_slot + 1, st);
  return dsp_block_update(e->blk[k], e->rule, e->ys[k], lr, e->s * lr, e->beta, e->wd, apply_update(e, k, n) ? 1 : 0,
                          loss_slot + 1, st);
}

// the blocks of device j at step n on its step stream (forked block streams if `forked`)
int issue_device(dsp_engine* e, int j, int64_t n, bool forked) {
  cudaStream_t ds = e->dstream[j];
  if (!forked) {
    for (int k = 0; k < e->K; ++k)
      if (e->dj[k] == j) DSP_TRY(issue_block(e, k, n, ds));
    return DSP_OK;
  }
  ENG_CUDA(cudaEventRecord(e->fork_ev[j], ds));
  for (int k = 0; k < e->K; ++k) {
    if (e->dj[k] != j) continue;
    ENG_CUDA(cudaStreamWaitEvent(e->bstream[k], e->fork_ev[j], 0));
    DSP_TRY(issue_block(e, k, n, e->bstream[k]));
    ENG_CUDA(cudaEventRecord(e->join_ev[k], e->bstream[k]));
  }
  for (int k = 0; k < e->K; ++k)
    if (e->dj[k] == j) ENG_CUDA(cudaStreamWaitEvent(ds, e->join_ev[k], 0));
  return DSP_OK;
}

int run_device_step(dsp_engine* e, int j, int64_t n) {
  if (!e->cfg.use_graphs || n < e->horizon) return issue_device(e, j, n, false);
  Phase& P = e->phases[j][n % e->R];
  std::vector<double> lr;
  std::vector<int> ap;
  for (int k = 0; k < e->K; ++k) {
    if (e->dj[k] != j) continue;
    lr.push_back(lr_at(e, n));
    ap.push_back(apply_update(e, k, n) ? 1 : 0);
  }
  if (P.exec == nullptr || P.lr != lr || P.apply != ap) {
    if (P.exec != nullptr) {
      ENG_CUDA(cudaGraphExecDestroy(P.exec));
      P.exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    ENG_CUDA(cudaStreamBeginCapture(e->dstream[j], cudaStreamCaptureModeThreadLocal));
    const int rc = issue_device(e, j, n, true);
    const cudaError_t ce = cudaStreamEndCapture(e->dstream[j], &g);
    if (rc != DSP_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    ENG_CUDA(ce);
    const cudaError_t ie = cudaGraphInstantiateWithFlags(&P.exec, g, 0);
    cudaGraphDestroy(g);
    ENG_CUDA(ie);
    P.lr = lr;
    P.apply = ap;
  }
  ENG_CUDA(cudaGraphLaunch(P.exec, e->dstream[j]));
  return DSP_OK;
}

// NonFiniteError (tensor.py:34-37, optim.py:53 / 89) at the sync point ending dsp_run
int check_nonfinite(dsp_engine* e) {
  for (int k = 0; k < e->K; ++k) {
    int f = 0;
    ENG_CUDA(cudaSetDevice(dev_of(e, k)));
    DSP_TRY(dsp_block_nonfinite(e->blk[k], 0, &f, e->dstream[e->dj[k]]));
    if (f & DSP_NONFINITE_LOSS)
      return set_error(DSP_E_NONFINITE, "non-finite values in softmax_xent (block %d, by step %lld)", k,
                       (long long)e->steps - 1);
    if (f & DSP_NONFINITE_GRAD)
      return set_error(DSP_E_NONFINITE, "non-finite gradient in %s (block %d, by step %lld)",
                       e->rule == DSP_RULE_SGD ? "sgd_step" : "sum_step", k, (long long)e->steps - 1);
  }
  return DSP_OK;
}

int sync_all(dsp_engine* e) {
  for (int j = 0; j < e->ndev; ++j) {
    ENG_CUDA(cudaSetDevice(e->devs[j]));
    ENG_CUDA(cudaStreamSynchronize(e->dstream[j]));
  }
  return DSP_OK;
}

void drop_graphs(dsp_engine* e) {
  for (int j = 0; j < e->ndev; ++j)
    for (auto& P : e->phases[j])
      if (P.exec) {
        cudaGraphExecDestroy(P.exec);
        P.exec = nullptr;
      }
}

}  // namespace

extern "C" int dsp_create(const dsp_config_t* cfg, dsp_engine_t** out) {
  if (!cfg || !out) return set_error(DSP_E_INVALID, "dsp_create: null argument");
  DSP_TRY(validate(*cfg));
  dsp_engine* e = new dsp_engine();
  *out = nullptr;
  e->cfg = *cfg;
  e->K = cfg->K;
  e->B = cfg->batch;
  e->D = cfg->in_c * cfg->in_h * cfg->in_w;
  const int K = e->K;
  // device map
  e->ndev = 0;
  for (int k = 0; k < K; ++k) {
    const int d = cfg->multi_device ? cfg->device_of_block[k] : cfg->device;
    int j = 0;
    while (j < e->ndev && e->devs[j] != d) ++j;
    if (j == e->ndev) e->devs[e->ndev++] = d;
    e->dj[k] = j;
  }
  for (int k = 0; k < K; ++k)
    for (int nb : {k - 1, k + 1})
      if (nb >= 0 && nb < K && e->dj[nb] != e->dj[k]) e->nbr[e->dj[k]][e->dj[nb]] = true;
  auto fail = [&](int rc) {
    dsp_destroy(e);
    return rc;
  };
  // peer access along every cross-device FIFO edge (the producer stores into the consumer's ring)
  for (int k = 0; k + 1 < K; ++k) {
    const int a = dev_of(e, k), b = dev_of(e, k + 1);
    if (a == b) continue;
    for (auto pr : {std::make_pair(a, b), std::make_pair(b, a)}) {
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, pr.first, pr.second) != cudaSuccess || !ok)
        return fail(set_error(DSP_E_CUDA, "dsp_create: device %d cannot access device %d (peer access)", pr.first,
                              pr.second));
      if (cudaSetDevice(pr.first) != cudaSuccess) return fail(set_error(DSP_E_CUDA, "cudaSetDevice failed"));
      const cudaError_t pe = cudaDeviceEnablePeerAccess(pr.second, 0);
      if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (pe != cudaSuccess) return fail(check(pe, "cudaDeviceEnablePeerAccess"));
    }
  }
  int total_layers = 0;
  for (int k = 0; k < K; ++k) total_layers += cfg->n_layers[k];
  e->layers.assign(cfg->layers, cfg->layers + total_layers);
  e->cfg.layers = e->layers.data();
  for (int k = 0; k < K; ++k) e->cum_p[k + 1] = e->cum_p[k] + cfg->p[k];
  e->q[0] = 0;
  for (int k = 1; k < K; ++k) e->q[k] = cfg->m[k - 1] - cfg->p[k - 1] - cfg->m[k];
  // ring depth: longer than every packet's lifetime in steps
  int life = cfg->m[0] + 1;
  for (int k = 0; k + 1 < K; ++k) life = std::max(life, cfg->p[k] + cfg->m[k + 1] + 1);
  for (int k = 1; k < K; ++k) life = std::max(life, e->q[k] + 1);
  life = std::max(life, e->cum_p[K - 1] + cfg->m[K - 1] + 1);  // labels of the last block's stale batch
  e->R = life + 1;
  int maxm = 0, maxp = 0, maxq = 0;
  for (int k = 0; k < K; ++k) {
    maxm = std::max(maxm, cfg->m[k]);
    maxp = std::max(maxp, cfg->p[k]);
    maxq = std::max(maxq, e->q[k]);
  }
  e->horizon = e->cum_p[K - 1] + maxm + maxp + maxq + 1;  // no zero packet is read from here on
  static const char* tw_env = getenv("DSP_B200_TWIN");
  int off = 0;
  int64_t max_act[kMaxDev] = {};
  for (int k = 0; k < K; ++k) {
    if (cudaSetDevice(dev_of(e, k)) != cudaSuccess) return fail(set_error(DSP_E_CUDA, "cudaSetDevice failed"));
    int rc = dsp_block_create(e->layers.data() + off, cfg->n_layers[k], e->B, cfg->dtype, k == K - 1, &e->blk[k]);
    if (rc != DSP_OK) return fail(rc);
    off += cfg->n_layers[k];
    e->nparam[k] = dsp_block_param_count(e->blk[k]);
    e->in_elems[k] = dsp_block_in_elems(e->blk[k]);
    e->out_elems[k] = dsp_block_out_elems(e->blk[k]);
    max_act[e->dj[k]] = std::max(max_act[e->dj[k]], e->in_elems[k]);
    if ((rc = dmalloc(&e->ws[k], dsp_block_workspace_bytes(e->blk[k]))) != DSP_OK) return fail(rc);
    if ((rc = dmalloc(&e->params[k], sizeof(float) * e->nparam[k], true)) != DSP_OK) return fail(rc);
    if ((rc = dmalloc(&e->grads[k], sizeof(float) * e->nparam[k], true)) != DSP_OK) return fail(rc);
    // optimizer state: ys (SUM) or the Adam state, whichever rule dsp_set_optimizer picks
    if ((rc = dmalloc(&e->ys[k], std::max(sizeof(float) * e->nparam[k], DSP_ADAM_STATE_BYTES(e->nparam[k])), true)) !=
        DSP_OK)
      return fail(rc);
  }
  for (int j = 0; j < e->ndev; ++j) {
    if (cudaSetDevice(e->devs[j]) != cudaSuccess) return fail(set_error(DSP_E_CUDA, "cudaSetDevice failed"));
    if (cudaStreamCreateWithFlags(&e->dstream[j], cudaStreamNonBlocking) != cudaSuccess) return fail(DSP_E_CUDA);
    if (cudaEventCreateWithFlags(&e->fork_ev[j], cudaEventDisableTiming) != cudaSuccess) return fail(DSP_E_CUDA);
    for (int p = 0; p < 2; ++p)
      if (cudaEventCreateWithFlags(&e->done_ev[j][p], cudaEventDisableTiming) != cudaSuccess) return fail(DSP_E_CUDA);
    e->phases[j].resize(e->R);
  }
  for (int k = 0; k < K; ++k) {
    if (cudaSetDevice(dev_of(e, k)) != cudaSuccess) return fail(set_error(DSP_E_CUDA, "cudaSetDevice failed"));
    cudaStream_t ds = e->dstream[e->dj[k]];
    if (cudaStreamCreateWithFlags(&e->bstream[k], cudaStreamNonBlocking) != cudaSuccess) return fail(DSP_E_CUDA);
    if (cudaEventCreateWithFlags(&e->join_ev[k], cudaEventDisableTiming) != cudaSuccess) return fail(DSP_E_CUDA);
    int rc = dsp_block_bind(e->blk[k], e->ws[k], e->params[k], e->grads[k], ds);
    if (rc != DSP_OK) return fail(rc);
    // forward twins when a device holds few blocks (engine_b200.use_twins; DSP_B200_TWIN=0/1)
    int on_dev = 0;
    for (int k2 = 0; k2 < K; ++k2) on_dev += e->dj[k2] == e->dj[k];
    const bool twins = tw_env ? tw_env[0] == '1' : on_dev <= 8;
    if (k < K - 1 && twins) {
      const int off_k = (int)(std::accumulate(cfg->n_layers, cfg->n_layers + k, 0));
      if ((rc = dsp_block_create(e->layers.data() + off_k, cfg->n_layers[k], e->B, cfg->dtype, 0, &e->twin[k])) !=
          DSP_OK)
        return fail(rc);
      if ((rc = dmalloc(&e->tws[k], dsp_block_workspace_bytes(e->twin[k]))) != DSP_OK) return fail(rc);
      if ((rc = dsp_block_bind(e->twin[k], e->tws[k], e->params[k], e->grads[k], ds)) != DSP_OK) return fail(rc);
      if ((rc = dsp_block_share_weights(e->twin[k], e->blk[k])) != DSP_OK) return fail(rc);
      if (cudaStreamCreateWithFlags(&e->fstream[k], cudaStreamNonBlocking) != cudaSuccess) return fail(DSP_E_CUDA);
      if (cudaEventCreateWithFlags(&e->fev_fork[k], cudaEventDisableTiming) != cudaSuccess) return fail(DSP_E_CUDA);
      if (cudaEventCreateWithFlags(&e->fev_join[k], cudaEventDisableTiming) != cudaSuccess) return fail(DSP_E_CUDA);
    }
  }
  const int R = e->R;
  const size_t esz = cfg->dtype == DSP_DTYPE_F32 ? 4 : 2;
  int rc = DSP_OK;
  for (int k = 0; k < K && rc == DSP_OK; ++k) {
    if (k < K - 1) {  // block k's output packets live on block k+1's device
      rc = check(cudaSetDevice(dev_of(e, k + 1)), "cudaSetDevice");
      e->ring_out[k].resize(R);
      for (int r = 0; r < R && rc == DSP_OK; ++r) rc = dmalloc(&e->ring_out[k][r], esz * e->out_elems[k], true);
    }
    if (k > 0 && rc == DSP_OK) {  // block k's input gradients live on block k-1's device
      rc = check(cudaSetDevice(dev_of(e, k - 1)), "cudaSetDevice");
      e->ring_gin[k].resize(R);
      for (int r = 0; r < R && rc == DSP_OK; ++r) rc = dmalloc(&e->ring_gin[k][r], esz * e->in_elems[k], true);
    }
  }
  for (int j = 0; j < e->ndev && rc == DSP_OK; ++j) {
    rc = check(cudaSetDevice(e->devs[j]), "cudaSetDevice");
    // zero packets: a device's blocks read them as inputs and as upstream gradients
    int64_t mx = max_act[j];
    for (int k = 0; k + 1 < K; ++k)
      if (e->dj[k] == j) mx = std::max(mx, e->out_elems[k]);
    if (rc == DSP_OK) rc = dmalloc(&e->zero_act[j], esz * mx, true);
    if (rc == DSP_OK) rc = dmalloc(&e->slots[j], sizeof(float) * (size_t)R * K * 2, true);
  }
  if (rc == DSP_OK) rc = check(cudaSetDevice(dev_of(e, 0)), "cudaSetDevice");
  e->ring_in.resize(R);
  for (int r = 0; r < R && rc == DSP_OK; ++r) rc = dmalloc(&e->ring_in[r], esz * e->in_elems[0], true);
  for (int i = 0; i < 2 && rc == DSP_OK; ++i) rc = dmalloc(&e->xdev[i], sizeof(float) * (size_t)e->B * e->D);
  if (rc == DSP_OK) rc = check(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  for (int i = 0; i < 2 && rc == DSP_OK; ++i) {
    rc = check(cudaMallocHost((void**)&e->pin_x[i], sizeof(float) * (size_t)e->B * e->D), "cudaMallocHost");
    if (rc == DSP_OK) rc = check(cudaMallocHost((void**)&e->pin_l[i], sizeof(int64_t) * e->B), "cudaMallocHost");
    if (rc == DSP_OK) rc = check(cudaEventCreateWithFlags(&e->pin_ev[i], cudaEventDisableTiming), "cudaEventCreate");
  }
  if (rc == DSP_OK) rc = check(cudaSetDevice(dev_of(e, K - 1)), "cudaSetDevice");
  e->ring_lab.resize(R);
  for (int r = 0; r < R && rc == DSP_OK; ++r) rc = dmalloc(&e->ring_lab[r], sizeof(int64_t) * e->B, true);
  if (rc == DSP_OK) rc = dmalloc(&e->zero_lab, sizeof(int64_t) * e->B, true);
  if (rc == DSP_OK) rc = check(cudaStreamCreateWithFlags(&e->lab_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  for (int i = 0; i < 2 && rc == DSP_OK; ++i)
    rc = check(cudaEventCreateWithFlags(&e->lab_ev[i], cudaEventDisableTiming), "cudaEventCreate");
  if (rc != DSP_OK) return fail(rc);
  for (int j = 0; j < e->ndev; ++j) {
    if (cudaSetDevice(e->devs[j]) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
      return fail(set_error(DSP_E_CUDA, "dsp_create: device sync failed"));
  }
  *out = e;
  return DSP_OK;
}

extern "C" size_t dsp_param_count(dsp_engine_t* e, int k) {
  return (e && k >= 0 && k < e->K) ? (size_t)e->nparam[k] : 0;
}

extern "C" int dsp_set_params(dsp_engine_t* e, int k, const void* src, size_t n, int on_device) {
  if (!e || k < 0 || k >= e->K || !src) return set_error(DSP_E_INVALID, "dsp_set_params: bad arguments");
  if ((int64_t)n != e->nparam[k])
    return set_error(DSP_E_INVALID, "dsp_set_params: block %d has %lld params, got %zu", k, (long long)e->nparam[k], n);
  ENG_CUDA(cudaSetDevice(dev_of(e, k)));
  cudaStream_t st = e->dstream[e->dj[k]];
  if (on_device) {
    ENG_CUDA(cudaMemcpyAsync(e->params[k], src, sizeof(float) * n, cudaMemcpyDefault, st));
  } else {
    std::vector<float> f(n);
    const double* d = static_cast<const double*>(src);
    for (size_t i = 0; i < n; ++i) f[i] = (float)d[i];
    ENG_CUDA(cudaMemcpyAsync(e->params[k], f.data(), sizeof(float) * n, cudaMemcpyHostToDevice, st));
    ENG_CUDA(cudaStreamSynchronize(st));
  }
  // optimizer state follows the parameters (OptimizerState.for_params: ys_0 = x_0)
  // (Adam: m = v = 0, step counter 0)
  if (e->rule == DSP_RULE_ADAM)
    ENG_CUDA(cudaMemsetAsync(e->ys[k], 0, DSP_ADAM_STATE_BYTES(n), st));
  else
    ENG_CUDA(cudaMemcpyAsync(e->ys[k], e->params[k], sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
  DSP_TRY(dsp_block_pack(e->blk[k], st));
  ENG_CUDA(cudaStreamSynchronize(st));
  return DSP_OK;
}

extern "C" int dsp_get_params(dsp_engine_t* e, int k, double* dst, size_t n) {
  if (!e || k < 0 || k >= e->K || !dst) return set_error(DSP_E_INVALID, "dsp_get_params: bad arguments");
  if ((int64_t)n != e->nparam[k])
    return set_error(DSP_E_INVALID, "dsp_get_params: block %d has %lld params, got %zu", k, (long long)e->nparam[k], n);
  ENG_CUDA(cudaSetDevice(dev_of(e, k)));
  cudaStream_t st = e->dstream[e->dj[k]];
  std::vector<float> f(n);
  ENG_CUDA(cudaMemcpyAsync(f.data(), e->params[k], sizeof(float) * n, cudaMemcpyDeviceToHost, st));
  ENG_CUDA(cudaStreamSynchronize(st));
  for (size_t i = 0; i < n; ++i) dst[i] = f[i];
  return DSP_OK;
}

extern "C" int dsp_set_optimizer(dsp_engine_t* e, int rule, double beta, double s, double wd, double base_lr,
                                 const int64_t* decay_steps, const double* factors, int n_decay) {
  if (!e) return set_error(DSP_E_INVALID, "dsp_set_optimizer: null engine");
  if (rule != DSP_RULE_SGD && rule != DSP_RULE_SUM && rule != DSP_RULE_ADAM)
    return set_error(DSP_E_INVALID, "dsp_set_optimizer: bad rule %d", rule);
  if (n_decay < 0 || (n_decay > 0 && (!decay_steps || !factors)))
    return set_error(DSP_E_INVALID, "dsp_set_optimizer: bad decay list");
  if (rule != e->rule) {  // re-initialise the optimizer state for the new rule (for_params)
    for (int k = 0; k < e->K; ++k) {
      const size_t n = (size_t)e->nparam[k];
      ENG_CUDA(cudaSetDevice(dev_of(e, k)));
      cudaStream_t st = e->dstream[e->dj[k]];
      if (rule == DSP_RULE_ADAM)
        ENG_CUDA(cudaMemsetAsync(e->ys[k], 0, DSP_ADAM_STATE_BYTES(n), st));
      else if (n)
        ENG_CUDA(cudaMemcpyAsync(e->ys[k], e->params[k], sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
    }
    DSP_TRY(sync_all(e));
  }
  e->rule = rule;
  e->beta = beta;
  e->s = s;
  e->wd = wd;
  e->base_lr = base_lr;
  e->decays.clear();
  for (int i = 0; i < n_decay; ++i) e->decays.push_back({decay_steps[i], factors[i]});
  drop_graphs(e);  // captured steps baked the old constants in
  return DSP_OK;
}

// Host batch -> pinned staging copy on several threads: one thread moves ~10 GB/s, so a 154 MB
// ImageNet-shaped batch took ~16 ms of the host's per-step issue loop (DSP_B200_COPY_THREADS).
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  static const int nt = [] {
    const char* v = getenv("DSP_B200_COPY_THREADS");
    const int hw = (int)std::thread::hardware_concurrency();
    return v ? std::max(1, atoi(v)) : std::max(1, std::min(8, hw / 2));
  }();
  const size_t min_chunk = size_t(8) << 20;
  const int t = (int)std::min<size_t>((size_t)nt, std::max<size_t>(1, bytes / min_chunk));
  if (t <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes / t + 4095) & ~size_t(4095);
  std::vector<std::thread> th;
  for (int k = 1; k < t; ++k) {
    const size_t off = per * k;
    if (off >= bytes) break;
    th.emplace_back([=] { memcpy((char*)dst + off, (const char*)src + off, std::min(per, bytes - off)); });
  }
  memcpy(dst, src, std::min(per, bytes));
  for (auto& x : th) x.join();
}

extern "C" int dsp_run(dsp_engine_t* e, int n_steps, const float* x, const int64_t* labels) {
  if (!e || n_steps < 0 || (n_steps > 0 && (!x || !labels))) return set_error(DSP_E_INVALID, "dsp_run: bad arguments");
  const size_t xb = sizeof(float) * (size_t)e->B * e->D, lb = sizeof(int64_t) * e->B;
  const int K = e->K, j0 = e->dj[0], jl = e->dj[K - 1];
  for (int i = 0; i < n_steps; ++i) {
    const int64_t n = e->steps;
    const int64_t* lab = labels + (size_t)i * e->B;
    for (int b = 0; b < e->B; ++b)
      if (lab[b] < 0 || lab[b] >= e->cfg.num_classes)
        return set_error(DSP_E_INVALID, "dsp_run: label out of range [0, %d) at step %lld", e->cfg.num_classes,
                         (long long)n);
    // batch n: host -> pinned slot -> device staging -> packed ring slot (block 0's input) on
    // block 0's copy stream, the labels on the last block's, so they overlap step n-1. Safe once
    // step n-2 is done: ring slot n mod R was last read by step n-R+m_0 (labels:
    // n-R+cum_p[K-1]+m_{K-1}) <= n-2.
    const int pi = (int)(n & 1);
    ENG_CUDA(cudaEventSynchronize(e->pin_ev[pi]));  // batch n-2's copies out of this pinned slot are done
    ENG_CUDA(cudaEventSynchronize(e->lab_ev[pi]));
    par_memcpy(e->pin_x[pi], x + (size_t)i * e->B * e->D, xb);
    memcpy(e->pin_l[pi], lab, lb);
    const int slot = (int)(n % e->R);
    ENG_CUDA(cudaSetDevice(e->devs[j0]));
    if (n >= 2) ENG_CUDA(cudaStreamWaitEvent(e->copy_stream, e->done_ev[j0][pi], 0));  // step n-2 done
    ENG_CUDA(cudaMemcpyAsync(e->xdev[pi], e->pin_x[pi], xb, cudaMemcpyHostToDevice, e->copy_stream));
    DSP_TRY(dsp_pack_input(e->xdev[pi], e->ring_in[slot], e->B, e->cfg.in_c, e->cfg.in_h, e->cfg.in_w,
                           (e->cfg.in_c + 7) / 8 * 8, e->cfg.dtype, 1, e->copy_stream));
    ENG_CUDA(cudaEventRecord(e->pin_ev[pi], e->copy_stream));
    ENG_CUDA(cudaSetDevice(e->devs[jl]));
    if (n >= 2) ENG_CUDA(cudaStreamWaitEvent(e->lab_stream, e->done_ev[jl][pi], 0));
    ENG_CUDA(cudaMemcpyAsync(e->ring_lab[slot], e->pin_l[pi], lb, cudaMemcpyHostToDevice, e->lab_stream));
    ENG_CUDA(cudaEventRecord(e->lab_ev[pi], e->lab_stream));
    for (int j = 0; j < e->ndev; ++j) {
      ENG_CUDA(cudaSetDevice(e->devs[j]));
      cudaStream_t ds = e->dstream[j];
      if (j == j0) ENG_CUDA(cudaStreamWaitEvent(ds, e->pin_ev[pi], 0));
      if (j == jl) ENG_CUDA(cudaStreamWaitEvent(ds, e->lab_ev[pi], 0));
      if (n >= 1)  // the neighbours' step n-1 (packets written / slots read)
        for (int i2 = 0; i2 < e->ndev; ++i2)
          if (e->nbr[j][i2]) ENG_CUDA(cudaStreamWaitEvent(ds, e->done_ev[i2][pi ^ 1], 0));
      DSP_TRY(run_device_step(e, j, n));
      // this device's blocks' loss / grad-norm rows -> its pinned host log (asynchronous)
      const int64_t row = n;
      if (row / dsp_engine::LOG_CHUNK >= (int64_t)e->host_log[j].size()) {
        float* chunk = nullptr;
        ENG_CUDA(cudaMallocHost((void**)&chunk, sizeof(float) * dsp_engine::LOG_CHUNK * K * 2));
        e->host_log[j].push_back(chunk);
      }
      float* dst = e->host_log[j][row / dsp_engine::LOG_CHUNK] + (row % dsp_engine::LOG_CHUNK) * K * 2;
      ENG_CUDA(cudaMemcpyAsync(dst, e->slots[j] + (size_t)slot * K * 2, sizeof(float) * K * 2,
                               cudaMemcpyDeviceToHost, ds));
      ENG_CUDA(cudaEventRecord(e->done_ev[j][pi], ds));
    }
    e->steps = n + 1;
  }
  DSP_TRY(sync_all(e));
  ENG_CUDA(cudaSetDevice(e->devs[j0]));
  ENG_CUDA(cudaStreamSynchronize(e->copy_stream));
  ENG_CUDA(cudaSetDevice(e->devs[jl]));
  ENG_CUDA(cudaStreamSynchronize(e->lab_stream));
  return check_nonfinite(e);
}

extern "C" int64_t dsp_steps_done(dsp_engine_t* e) { return e ? e->steps : -1; }

extern "C" int dsp_read_log(dsp_engine_t* e, dsp_log_record_t* recs, size_t cap, size_t* n) {
  if (!e || !n || (cap > 0 && !recs)) return set_error(DSP_E_INVALID, "dsp_read_log: bad arguments");
  DSP_TRY(sync_all(e));
  const size_t total = (size_t)e->steps * e->K;
  *n = total;
  size_t w = 0;
  for (int64_t s = 0; s < e->steps && w < cap; ++s) {
    for (int k = 0; k < e->K && w < cap; ++k, ++w) {
      const float* row = e->host_log[e->dj[k]][s / dsp_engine::LOG_CHUNK] + (s % dsp_engine::LOG_CHUNK) * e->K * 2;
      dsp_log_record_t& r = recs[w];
      r.step = s;
      r.block = k;
      r.batch_index = s - e->cum_p[k] - e->cfg.m[k];
      r.has_loss = k == e->K - 1;
      r.loss = r.has_loss ? (double)row[k * 2] : NAN;
      r.grad_norm = std::sqrt((double)row[k * 2 + 1]);
    }
  }
  return DSP_OK;
}

extern "C" void dsp_destroy(dsp_engine_t* e) {
  if (!e) return;
  for (int j = 0; j < e->ndev; ++j) {
    cudaSetDevice(e->devs[j]);
    if (e->dstream[j]) cudaStreamSynchronize(e->dstream[j]);
  }
  drop_graphs(e);
  for (int k = 0; k < DSP_MAX_BLOCKS; ++k) {
    if (k < e->K) cudaSetDevice(dev_of(e, k));
    if (e->blk[k]) dsp_block_destroy(e->blk[k]);
    cudaFree(e->ws[k]);
    if (e->twin[k]) dsp_block_destroy(e->twin[k]);
    if (e->tws[k]) cudaFree(e->tws[k]);
    if (e->fstream[k]) cudaStreamDestroy(e->fstream[k]);
    if (e->fev_fork[k]) cudaEventDestroy(e->fev_fork[k]);
    if (e->fev_join[k]) cudaEventDestroy(e->fev_join[k]);
    cudaFree(e->params[k]);
    cudaFree(e->grads[k]);
    cudaFree(e->ys[k]);
    for (void* p : e->ring_out[k]) cudaFree(p);
    for (void* p : e->ring_gin[k]) cudaFree(p);
    if (e->bstream[k]) cudaStreamDestroy(e->bstream[k]);
    if (e->join_ev[k]) cudaEventDestroy(e->join_ev[k]);
  }
  for (void* p : e->ring_in) cudaFree(p);
  for (int64_t* p : e->ring_lab) cudaFree(p);
  cudaFree(e->zero_lab);
  if (e->copy_stream) cudaStreamSynchronize(e->copy_stream);
  if (e->lab_stream) cudaStreamSynchronize(e->lab_stream);
  for (int i = 0; i < 2; ++i) {
    cudaFree(e->xdev[i]);
    if (e->pin_x[i]) cudaFreeHost(e->pin_x[i]);
    if (e->pin_l[i]) cudaFreeHost(e->pin_l[i]);
    if (e->pin_ev[i]) cudaEventDestroy(e->pin_ev[i]);
    if (e->lab_ev[i]) cudaEventDestroy(e->lab_ev[i]);
  }
  for (int j = 0; j < e->ndev; ++j) {
    cudaSetDevice(e->devs[j]);
    cudaFree(e->zero_act[j]);
    cudaFree(e->slots[j]);
    for (float* c : e->host_log[j]) cudaFreeHost(c);
    if (e->fork_ev[j]) cudaEventDestroy(e->fork_ev[j]);
    for (int p = 0; p < 2; ++p)
      if (e->done_ev[j][p]) cudaEventDestroy(e->done_ev[j][p]);
    if (e->dstream[j]) cudaStreamDestroy(e->dstream[j]);
  }
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  if (e->lab_stream) cudaStreamDestroy(e->lab_stream);
  delete e;
}

extern "C" int dsp_set_adam(dsp_engine_t* e, double beta1, double beta2, double eps) {
  if (!e) return set_error(DSP_E_INVALID, "dsp_set_adam: null engine");
  if (!(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0) || !(eps > 0.0))
    return set_error(DSP_E_INVALID, "dsp_set_adam: bad hyper-parameters");
  e->adam_b1 = beta1;
  e->adam_b2 = beta2;
  e->adam_eps = eps;
  drop_graphs(e);  // captured steps baked the old constants in
  return DSP_OK;
}
