// abi.cu -- host side of libtacsnn: the C ABI declared in include/tacsnn.h.
// Validation, weight preparation, engine selection and launch on the caller's
// stream.  No device allocation; no exception crosses the ABI.
#include <cuda_runtime.h>

#include <cmath>
#include <map>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tacsnn.h"
#include "layer.cuh"
#include "tc.cuh"

namespace {

thread_local std::string g_detail;
thread_local int g_launches = 0;

tac_status fail(tac_status st, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
tac_status fail(tac_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_detail = buf;
  return st;
}

struct Geo {
  int Ho, Wo, Hq, Wq, G, T_out, nsteps, wpr_in, wpr_out, K;
  int K_last;  // frames of the last group (== K unless partial_last_group and K does not divide T)
  long long in_st, in_sb, out_st, out_sb;
};

tac_status check(const tac_conv_lif_desc *d, Geo *g) {
  if (!d) return fail(TAC_ERR_NULL, "desc is NULL");
  if (d->T < 1) return fail(TAC_ERR_SHAPE, "T=%d < 1", d->T);
  if (d->B < 1) return fail(TAC_ERR_SHAPE, "B=%d < 1", d->B);
  if (d->C_in < 1) return fail(TAC_ERR_SHAPE, "C_in=%d < 1", d->C_in);
  if (d->H < 1 || d->W < 1) return fail(TAC_ERR_SHAPE, "H=%d, W=%d must be >= 1", d->H, d->W);
  if (d->C_out < 1) return fail(TAC_ERR_SHAPE, "C_out=%d < 1", d->C_out);
  if (d->R < 1 || d->S < 1) return fail(TAC_ERR_SHAPE, "R=%d, S=%d must be >= 1", d->R, d->S);
  if (d->stride < 1) return fail(TAC_ERR_SHAPE, "stride=%d < 1", d->stride);
  if (d->pad < 0) return fail(TAC_ERR_SHAPE, "pad=%d < 0", d->pad);
  if (d->mode < 0 || d->mode > 2) return fail(TAC_ERR_PARAM, "mode=%d not in {0,1,2}", d->mode);
  if (d->reset < 0 || d->reset > 2) return fail(TAC_ERR_PARAM, "reset=%d not in {0,1,2}", d->reset);
  if (d->engine < 0 || d->engine > 2) return fail(TAC_ERR_PARAM, "engine=%d not in {0,1,2}", d->engine);
  if (d->out_pool != 1 && d->out_pool != 2)
    return fail(TAC_ERR_PARAM, "out_pool=%d not in {1,2}", d->out_pool);
  if (!std::isfinite(d->beta)) return fail(TAC_ERR_NONFINITE, "beta is not finite");
  if (!std::isfinite(d->v_th)) return fail(TAC_ERR_NONFINITE, "v_th is not finite");
  if (!std::isfinite(d->v_reset)) return fail(TAC_ERR_NONFINITE, "v_reset is not finite");
  if (!(d->beta > 0.f && d->beta < 1.f))
    return fail(TAC_ERR_PARAM, "beta=%g not in (0,1) (PAPER.md:105)", (double)d->beta);
  if (!(d->v_th > 0.f)) return fail(TAC_ERR_PARAM, "v_th=%g must be > 0", (double)d->v_th);
  const int K = d->mode == TAC_MODE_DENSE ? 1 : d->K;
  if (K < 1 || (d->T % K != 0 && d->partial_last_group != 1))
    return fail(TAC_ERR_K_NOT_DIVIDING_T, "K=%d must be >= 1 and divide T=%d (PAPER.md:444)",
                d->K, d->T);
  if (K > tacsnn::kMaxK) return fail(TAC_ERR_UNSUPPORTED, "K=%d > %d", K, tacsnn::kMaxK);
  const int Ho = (d->H + 2 * d->pad - d->R) / d->stride + 1;
  const int Wo = (d->W + 2 * d->pad - d->S) / d->stride + 1;
  if (d->H + 2 * d->pad < d->R || Ho < 1)
    return fail(TAC_ERR_SHAPE, "output height H'=(H+2pad-R)/stride+1 < 1");
  if (d->W + 2 * d->pad < d->S || Wo < 1)
    return fail(TAC_ERR_SHAPE, "output width W'=(W+2pad-S)/stride+1 < 1");
  if (d->out_pool == 2 && (Ho < 2 || Wo < 2))
    return fail(TAC_ERR_SHAPE, "out_pool=2 needs H', W' >= 2 (H'=%d, W'=%d)", Ho, Wo);
  if ((long long)d->W * d->C_in > (1LL << 30) || (long long)Wo * d->C_out > (1LL << 30))
    return fail(TAC_ERR_SHAPE, "row too wide");
  if (d->in_stride_t < 0 || d->in_stride_b < 0 || d->out_stride_t < 0 || d->out_stride_b < 0)
    return fail(TAC_ERR_SHAPE, "negative stride");
  if (d->input_kind != TAC_INPUT_SPIKES && d->input_kind != TAC_INPUT_REAL)
    return fail(TAC_ERR_PARAM, "input_kind=%d not in {0,1}", d->input_kind);
  if (d->partial_last_group != 0 && d->partial_last_group != 1)
    return fail(TAC_ERR_PARAM, "partial_last_group=%d not in {0,1}", d->partial_last_group);
  if (d->agg_weights && d->mode != TAC_MODE_DENSE)
    for (int j = 0; j < K; ++j)
      if (!std::isfinite(d->agg_weights[j]))
        return fail(TAC_ERR_NONFINITE, "agg_weights[%d] is not finite", j);
  g->K = K;
  g->Ho = Ho;
  g->Wo = Wo;
  g->Hq = d->out_pool == 2 ? Ho / 2 : Ho;
  g->Wq = d->out_pool == 2 ? Wo / 2 : Wo;
  g->G = (d->T + K - 1) / K;
  g->K_last = d->T - (g->G - 1) * K;
  g->T_out = d->mode == TAC_MODE_TAC ? g->G : d->T;
  g->nsteps = d->mode == TAC_MODE_TACTP ? K : 1;
  g->wpr_in = (d->W * d->C_in + 31) / 32;
  g->wpr_out = (g->Wq * d->C_out + 31) / 32;
  // packed spikes: u32 words per (t, b) plane; REAL input: floats [H][W][C_in]
  const long long in_plane = d->input_kind == TAC_INPUT_REAL ? (long long)d->H * d->W * d->C_in
                                                              : (long long)d->H * g->wpr_in;
  const long long out_plane = (long long)g->Hq * g->wpr_out;
  g->in_sb = d->in_stride_b ? d->in_stride_b : in_plane;
  g->in_st = d->in_stride_t ? d->in_stride_t : in_plane * d->B;
  g->out_sb = d->out_stride_b ? d->out_stride_b : out_plane;
  g->out_st = d->out_stride_t ? d->out_stride_t : out_plane * d->B;
  if (g->in_sb < in_plane) return fail(TAC_ERR_SHAPE, "in_stride_b < one input plane");
  if (g->out_sb < out_plane) return fail(TAC_ERR_SHAPE, "out_stride_b < H_o*WPR_out");
  return TAC_OK;
}

// Prepared-weights buffer layout (device):
//   [0, simt_bytes)             SIMT fp32 weights [Cin][R][S][Cout]
//   [bias_off, +4*Cout)         fp32 bias
//   [tc_off, +tc bytes)         tcgen05 image (tc.cuh), when the shape qualifies
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct PrepLayout {
  size_t simt_off, bias_off, tc_off, tc_bytes, total;
};

PrepLayout prep_layout(const tac_conv_lif_desc *d) {
  PrepLayout L{};
  L.simt_off = 0;
  L.bias_off = align256((size_t)d->C_in * d->R * d->S * d->C_out * 4);
  L.tc_off = align256(L.bias_off + (size_t)d->C_out * 4);
  L.tc_bytes = tacsnn::tc_shape_ok(d) ? tacsnn::tc_weights_bytes(d) : 0;
  L.total = align256(L.tc_off + L.tc_bytes);
  return L;
}

// A layer with a short last group runs as two calls: the full groups (T1 = (G-1) K frames,
// group size K) and the last K' frames as one group of size K', chained through v_init /
// v_final in the workspace.  Each part has its own prepared image (the tcgen05 image
// depends on K), stored back to back.
bool is_split_call(const tac_conv_lif_desc *d, const Geo &g) {
  return d->partial_last_group == 1 && d->mode != TAC_MODE_DENSE && g.K_last != g.K;
}
tac_conv_lif_desc part_desc(const tac_conv_lif_desc *d, const Geo &g, bool last) {
  tac_conv_lif_desc p = *d;
  p.partial_last_group = 0;
  p.T = last ? g.K_last : (g.G - 1) * g.K;
  p.K = last ? g.K_last : g.K;
  p.in_stride_t = g.in_st;  // explicit: the parts keep the caller's layout
  p.in_stride_b = g.in_sb;
  p.out_stride_t = g.out_st;
  p.out_stride_b = g.out_sb;
  // the short group of K' frames aggregates with the last K' weights (reading R11)
  if (last && d->agg_weights && d->mode != TAC_MODE_DENSE) p.agg_weights = d->agg_weights + (g.K - g.K_last);
  // a short last group outside the tcgen05 envelope (K' not in {1,2,4,8}) runs on SIMT
  if (last && p.engine == TAC_ENGINE_TCGEN05 && !tacsnn::tc_supported(&p)) p.engine = TAC_ENGINE_AUTO;
  return p;
}
size_t prep_total(const tac_conv_lif_desc *d, const Geo &g) {
  if (!is_split_call(d, g)) return prep_layout(d).total;
  size_t n = 0;
  if (g.G > 1) {
    const tac_conv_lif_desc a = part_desc(d, g, false);
    n += prep_layout(&a).total;
  }
  const tac_conv_lif_desc b = part_desc(d, g, true);
  return n + prep_layout(&b).total;
}
int resolve_engine(const tac_conv_lif_desc *d);
size_t ws_total(const tac_conv_lif_desc *d, const Geo &g) {
  // a fully connected layer with few 128-sample tiles runs the two-phase tcgen05 FC
  // (GEMM units -> workspace -> LIF); without a workspace it runs fused
  if (!is_split_call(d, g))
    return (tacsnn::fc_is_fc(d) && resolve_engine(d) == TAC_ENGINE_TCGEN05) ? align256(tacsnn::fc_ws_bytes(d)) : 0;
  if (g.G == 1) return 0;
  return align256((size_t)d->B * g.Ho * g.Wo * d->C_out * 4) + align256((size_t)d->B * d->C_out * 4);
}

// Device-pointer check with a small per-thread cache of device allocation ranges
// (cuMemGetAddressRange): a launch-bound layer call then costs no
// cudaPointerGetAttributes round trips for buffers it has seen before (the torch
// caching allocator keeps its segments, so the ranges are stable).
struct Range {
  uintptr_t lo, hi;
};
thread_local Range g_ranges[32];
thread_local int g_nranges = 0, g_next_range = 0;
typedef int (*PFN_getAddressRange)(unsigned long long *, size_t *, unsigned long long);
PFN_getAddressRange address_range_fn() {
  static PFN_getAddressRange fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<PFN_getAddressRange>(f);
  }();
  return fn;
}
bool is_device_ptr(const void *p) {
  const uintptr_t u = reinterpret_cast<uintptr_t>(p);
  for (int i = 0; i < g_nranges; ++i)
    if (u >= g_ranges[i].lo && u < g_ranges[i].hi) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const bool dev = a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
  if (dev && a.type == cudaMemoryTypeDevice) {
    PFN_getAddressRange fn = address_range_fn();
    unsigned long long base = 0;
    size_t size = 0;
    if (fn && fn(&base, &size, (unsigned long long)u) == 0 && size) {
      g_ranges[g_next_range] = Range{(uintptr_t)base, (uintptr_t)base + size};
      g_next_range = (g_next_range + 1) % 32;
      if (g_nranges < 32) ++g_nranges;
    }
  }
  return dev;
}

// Fingerprint of the descriptor fields the prepared image depends on (tac_plan):
// FNV-1a over the geometry, the effective K, mode, beta / v_th bits, reset,
// input kind, the short-group size of a split call and the aggregation weights.
uint64_t fingerprint(const tac_conv_lif_desc *d, const Geo &g, bool split) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xFFu;
      h *= 1099511628211ull;
    }
  };
  uint32_t bits;
  mix((uint64_t)TACSNN_ABI_VERSION);
  mix((uint64_t)d->C_in); mix((uint64_t)d->C_out); mix((uint64_t)d->R); mix((uint64_t)d->S);
  mix((uint64_t)d->stride); mix((uint64_t)d->pad); mix((uint64_t)g.K); mix((uint64_t)d->mode);
  std::memcpy(&bits, &d->beta, 4); mix(bits);
  std::memcpy(&bits, &d->v_th, 4); mix(bits);
  mix((uint64_t)d->reset); mix((uint64_t)d->input_kind);
  mix(split ? (uint64_t)g.K_last : 0ull);
  mix(d->agg_weights && d->mode != TAC_MODE_DENSE ? 1ull : 0ull);
  if (d->agg_weights && d->mode != TAC_MODE_DENSE)
    for (int j = 0; j < g.K; ++j) {
      std::memcpy(&bits, &d->agg_weights[j], 4);
      mix(bits);
    }
  return h;
}

int resolve_engine(const tac_conv_lif_desc *d) {
  const bool tc = tacsnn::tc_supported(d);
  if (d->engine == TAC_ENGINE_SIMT) return TAC_ENGINE_SIMT;
  if (d->engine == TAC_ENGINE_TCGEN05) return tc ? TAC_ENGINE_TCGEN05 : -1;
  return tc ? TAC_ENGINE_TCGEN05 : TAC_ENGINE_SIMT;
}

}  // namespace

namespace tacsnn {
cudaError_t ensure_dyn_smem(const void *kern, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> done;  // (kernel, device) -> largest size set
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int &have = done[{kern, dev}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
}  // namespace tacsnn

extern "C" {

tac_status tac_desc_check(const tac_conv_lif_desc *desc) {
  g_detail.clear();
  Geo g;
  return check(desc, &g);
}

tac_status tac_out_shape(const tac_conv_lif_desc *desc, int32_t *T_out, int32_t *H_out,
                         int32_t *W_out, int32_t *wpr) {
  g_detail.clear();
  Geo g;
  tac_status st = check(desc, &g);
  if (st != TAC_OK) return st;
  if (T_out) *T_out = g.T_out;
  if (H_out) *H_out = g.Hq;
  if (W_out) *W_out = g.Wq;
  if (wpr) *wpr = g.wpr_out;
  return TAC_OK;
}

int32_t tac_select_engine(const tac_conv_lif_desc *desc) {
  g_detail.clear();
  Geo g;
  if (check(desc, &g) != TAC_OK) return -1;
  return resolve_engine(desc);
}

tac_status tac_weights_bytes(const tac_conv_lif_desc *desc, size_t *bytes) {
  g_detail.clear();
  Geo g;
  tac_status st = check(desc, &g);
  if (st != TAC_OK) return st;
  if (!bytes) return fail(TAC_ERR_NULL, "bytes is NULL");
  *bytes = prep_total(desc, g);
  return TAC_OK;
}

tac_status tac_workspace_bytes(const tac_conv_lif_desc *desc, size_t *bytes) {
  g_detail.clear();
  Geo g;
  tac_status st = check(desc, &g);
  if (st != TAC_OK) return st;
  if (!bytes) return fail(TAC_ERR_NULL, "bytes is NULL");
  *bytes = ws_total(desc, g);
  return TAC_OK;
}

tac_status tac_prepare_weights(const tac_conv_lif_desc *desc, const float *weight,
                               const float *bias, void *prepared, size_t bytes,
                               void *stream, tac_plan *plan) {
  g_detail.clear();
  Geo g;
  tac_status st = check(desc, &g);
  if (st != TAC_OK) return st;
  if (!weight) return fail(TAC_ERR_NULL, "weight is NULL");
  if (!plan) return fail(TAC_ERR_NULL, "plan is NULL");
  if (!prepared) return fail(TAC_ERR_NULL, "prepared is NULL");
  const size_t total = prep_total(desc, g);
  if (bytes < total) return fail(TAC_ERR_WORKSPACE, "prepared buffer %zu < %zu bytes", bytes, total);
  if ((uintptr_t)prepared % 256) return fail(TAC_ERR_ALIGN, "prepared must be 256-B aligned");
  if (!is_device_ptr(prepared)) return fail(TAC_ERR_PARAM, "prepared is not device memory");
  const int Co = desc->C_out, Ci = desc->C_in, R = desc->R, S = desc->S;
  const size_t nw = (size_t)Co * Ci * R * S;
  for (size_t i = 0; i < nw; ++i)
    if (!std::isfinite(weight[i])) return fail(TAC_ERR_NONFINITE, "weight[%zu] is not finite", i);
  if (bias)
    for (int i = 0; i < Co; ++i)
      if (!std::isfinite(bias[i])) return fail(TAC_ERR_NONFINITE, "bias[%d] is not finite", i);
  std::vector<unsigned char> img(total, 0);
  // one image per part (two when the last group is short): [full groups | last group]
  std::vector<tac_conv_lif_desc> parts;
  if (is_split_call(desc, g)) {
    if (g.G > 1) parts.push_back(part_desc(desc, g, false));
    parts.push_back(part_desc(desc, g, true));
  } else {
    parts.push_back(*desc);
  }
  size_t base = 0;
  uint32_t code = 0;  // fp16-path prescale exponent of each image part (plan->scale_code)
  int part = 0;
  for (const tac_conv_lif_desc &pd : parts) {
    const PrepLayout L = prep_layout(&pd);
    float *ws = reinterpret_cast<float *>(img.data() + base + L.simt_off);
    for (int co = 0; co < Co; ++co)
      for (int ci = 0; ci < Ci; ++ci)
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s)
            ws[((size_t)(ci * R + r) * S + s) * Co + co] = weight[((size_t)(co * Ci + ci) * R + r) * S + s];
    float *bs = reinterpret_cast<float *>(img.data() + base + L.bias_off);
    for (int co = 0; co < Co; ++co) bs[co] = bias ? bias[co] : 0.f;
    if (L.tc_bytes) {
      const int e = tacsnn::tc_prepare(&pd, weight, bias, img.data() + base + L.tc_off);
      code |= (uint32_t)(uint8_t)(int8_t)e << (8 * part);
    }
    base += L.total;
    ++part;
  }
  cudaError_t e = cudaMemcpyAsync(prepared, img.data(), total, cudaMemcpyHostToDevice,
                                  (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return fail(TAC_ERR_CUDA, "prepare copy: %s", cudaGetErrorString(e));
  plan->prepared = prepared;
  plan->bytes = total;
  plan->fingerprint = fingerprint(desc, g, is_split_call(desc, g));
  plan->abi_version = TACSNN_ABI_VERSION;
  plan->scale_code = (int32_t)code;
  return TAC_OK;
}

}  // extern "C"

namespace {
// fp16-path operand prescale exponent of image part `part` (0: the whole / full-group
// image, 1: the short last group's), as tac_prepare_weights recorded it
int plan_exp(const tac_plan *plan, int part) { return (int)(int8_t)((uint32_t)plan->scale_code >> (8 * part)); }

// Argument checks of one (non-split) launch, before anything is enqueued.
tac_status validate_call(const tac_conv_lif_desc *desc, const void *prepared, const void *input,
                         bool real, const float *v_init, const uint32_t *spikes_out,
                         const float *v_final, const uint32_t *counts, int *engine_out) {
  if ((desc->input_kind == TAC_INPUT_REAL) != real)
    return fail(TAC_ERR_PARAM, real ? "tac_conv_lif_forward_real needs input_kind = TAC_INPUT_REAL"
                                    : "input_kind = TAC_INPUT_REAL needs tac_conv_lif_forward_real");
  if (!prepared) return fail(TAC_ERR_NULL, "plan->prepared is NULL");
  if (!input) return fail(TAC_ERR_NULL, real ? "x_in is NULL" : "spikes_in is NULL");
  if (!spikes_out) return fail(TAC_ERR_NULL, "spikes_out is NULL");
  const int engine = resolve_engine(desc);
  if (engine < 0)
    return fail(TAC_ERR_UNSUPPORTED, "engine TCGEN05 cannot run this layer: %s",
                tacsnn::tc_unsupported_reason(desc));
  if ((uintptr_t)input % 4 || (uintptr_t)spikes_out % 4 || (uintptr_t)prepared % 256)
    return fail(TAC_ERR_ALIGN, "misaligned pointer");
  if (v_init && (uintptr_t)v_init % 16) return fail(TAC_ERR_ALIGN, "v_init must be 16-B aligned");
  if (v_final && (uintptr_t)v_final % 16) return fail(TAC_ERR_ALIGN, "v_final must be 16-B aligned");
  if (counts && (uintptr_t)counts % 4) return fail(TAC_ERR_ALIGN, "counts misaligned");
  const void *dev_ptrs[] = {prepared, input, spikes_out, v_init, v_final, counts};
  const char *names[] = {"prepared", real ? "x_in" : "spikes_in", "spikes_out", "v_init", "v_final",
                         "counts"};
  for (int i = 0; i < 6; ++i)
    if (dev_ptrs[i] && !is_device_ptr(dev_ptrs[i]))
      return fail(TAC_ERR_PARAM, "%s is not device memory", names[i]);
  *engine_out = engine;
  return TAC_OK;
}

// Enqueue one validated (non-split) call.
tac_status launch_call(const tac_conv_lif_desc *desc, const Geo &g, int engine, const void *prepared,
                       int yexp, const void *input, bool real, const float *v_init, uint32_t *spikes_out,
                       float *v_final, uint32_t *counts, void *stream, int *launches,
                       float *y_seq = nullptr, void *ws = nullptr, size_t ws_bytes = 0) {
  tacsnn::LayerParams p{};
  p.T = desc->T; p.B = desc->B; p.Cin = desc->C_in; p.H = desc->H; p.W = desc->W;
  p.Cout = desc->C_out; p.R = desc->R; p.S = desc->S; p.stride = desc->stride; p.pad = desc->pad;
  p.K = g.K; p.mode = desc->mode; p.reset = desc->reset; p.pool = desc->out_pool;
  p.Ho = g.Ho; p.Wo = g.Wo; p.Hq = g.Hq; p.Wq = g.Wq; p.G = g.G; p.nsteps = g.nsteps;
  p.T_out = g.T_out; p.wpr_in = g.wpr_in; p.wpr_out = g.wpr_out;
  p.in_st = g.in_st; p.in_sb = g.in_sb; p.out_st = g.out_st; p.out_sb = g.out_sb;
  p.v_th = desc->v_th; p.v_reset = desc->v_reset;
  const double beta = (double)desc->beta;
  p.decay = (float)(desc->mode == TAC_MODE_TAC ? std::pow(beta, (double)g.K) : beta);
  // A_k weights: beta^{K-1-j} or the learnable alpha_j
  const bool alpha = desc->agg_weights && desc->mode != TAC_MODE_DENSE;
  for (int j = 0; j < g.K; ++j)
    p.coef[j] = alpha ? desc->agg_weights[j] : (float)std::pow(beta, (double)(g.K - 1 - j));
  p.in = real ? nullptr : static_cast<const uint32_t *>(input);
  p.out = spikes_out; p.v_init = v_init; p.v_final = v_final; p.counts = counts;
  p.xin = real ? static_cast<const float *>(input) : nullptr;
  p.y_seq = y_seq;
  p.yscale_exp = yexp;
  p.ws = ws;
  p.ws_bytes = ws_bytes;
  const PrepLayout L = prep_layout(desc);
  const unsigned char *base = static_cast<const unsigned char *>(prepared);
  p.w = reinterpret_cast<const float *>(base + L.simt_off);
  p.bias = reinterpret_cast<const float *>(base + L.bias_off);
  int err = 0;
  if (engine == TAC_ENGINE_TCGEN05) {
    err = tacsnn::tc_launch(desc, p, base + L.tc_off, stream, launches);
  } else {
    err = tacsnn::launch_zero_outputs(p, stream, launches);
    if (!err) err = tacsnn::launch_simt_conv_lif(p, stream, launches);
  }
  if (err) return fail(TAC_ERR_CUDA, "launch failed: %s", cudaGetErrorString((cudaError_t)err));
  return TAC_OK;
}

// shared body of tac_conv_lif_forward / tac_conv_lif_forward_real: plan check, then
// one launch, or -- K not dividing T with partial_last_group -- the full groups and
// the short last group chained through the membrane state in the workspace (both
// parts validated before the first launch)
tac_status forward_impl(const tac_conv_lif_desc *desc, const tac_plan *plan, const void *input,
                        bool real, const float *v_init, uint32_t *spikes_out, float *v_final,
                        uint32_t *counts, void *ws, size_t ws_bytes, void *stream) {
  g_detail.clear();
  g_launches = 0;
  Geo g;
  tac_status st = check(desc, &g);
  if (st != TAC_OK) return st;
  if (!plan) return fail(TAC_ERR_NULL, "plan is NULL");
  if (plan->abi_version != TACSNN_ABI_VERSION)
    return fail(TAC_ERR_PARAM, "plan prepared by ABI version %d, library is %d", plan->abi_version,
                TACSNN_ABI_VERSION);
  const bool split = is_split_call(desc, g);
  if (plan->fingerprint != fingerprint(desc, g, split))
    return fail(TAC_ERR_PARAM, "plan was prepared for a different descriptor (C_in, C_out, kernel, "
                               "K, mode, beta, v_th, reset, input kind, short group or agg_weights "
                               "differ; see tac_plan)");
  const size_t need = prep_total(desc, g);
  if (plan->bytes < need) return fail(TAC_ERR_WORKSPACE, "plan image %zu < %zu bytes", plan->bytes, need);
  const void *prepared = plan->prepared;
  int launches = 0;
  if (!split) {
    int engine;
    st = validate_call(desc, prepared, input, real, v_init, spikes_out, v_final, counts, &engine);
    if (st != TAC_OK) return st;
    // optional workspace (two-phase tcgen05 FC layers); NULL runs the fused path
    const size_t wneed = ws_total(desc, g);
    if (ws && wneed) {
      if (ws_bytes < wneed) return fail(TAC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, wneed);
      if ((uintptr_t)ws % 256) return fail(TAC_ERR_ALIGN, "workspace must be 256-B aligned");
      if (!is_device_ptr(ws)) return fail(TAC_ERR_PARAM, "workspace is not device memory");
    }
    st = launch_call(desc, g, engine, prepared, plan_exp(plan, 0), input, real, v_init, spikes_out, v_final, counts, stream,
                     &launches, nullptr, wneed ? ws : nullptr, wneed ? ws_bytes : 0);
    if (st == TAC_OK) g_launches = launches;
    return st;
  }
  const tac_conv_lif_desc last = part_desc(desc, g, true);
  Geo gl;
  if ((st = check(&last, &gl)) != TAC_OK) return st;
  if (g.G == 1) {  // T < K: the whole sequence is one short group
    int engine;
    st = validate_call(&last, prepared, input, real, v_init, spikes_out, v_final, counts, &engine);
    if (st != TAC_OK) return st;
    st = launch_call(&last, gl, engine, prepared, plan_exp(plan, 0), input, real, v_init, spikes_out, v_final, counts, stream,
                     &launches);
    if (st == TAC_OK) g_launches = launches;
    return st;
  }
  if (!input || !spikes_out) return fail(TAC_ERR_NULL, "NULL buffer");
  if (!ws) return fail(TAC_ERR_NULL, "partial_last_group with K not dividing T needs a workspace");
  const size_t wneed = ws_total(desc, g);
  if (ws_bytes < wneed) return fail(TAC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, wneed);
  if ((uintptr_t)ws % 256) return fail(TAC_ERR_ALIGN, "workspace must be 256-B aligned");
  const tac_conv_lif_desc full = part_desc(desc, g, false);
  Geo gf;
  if ((st = check(&full, &gf)) != TAC_OK) return st;
  float *v_mid = static_cast<float *>(ws);
  uint32_t *cnt2 = reinterpret_cast<uint32_t *>(static_cast<unsigned char *>(ws) +
                                                align256((size_t)desc->B * g.Ho * g.Wo * desc->C_out * 4));
  const size_t esz = real ? sizeof(float) : sizeof(uint32_t);
  const void *in2 = static_cast<const unsigned char *>(input) + (size_t)full.T * g.in_st * esz;
  const int t_out1 = desc->mode == TAC_MODE_TAC ? g.G - 1 : full.T;
  uint32_t *out2 = spikes_out + (size_t)t_out1 * g.out_st;
  const void *prep2 = static_cast<const unsigned char *>(prepared) + prep_layout(&full).total;
  int eng1, eng2;
  if ((st = validate_call(&full, prepared, input, real, v_init, spikes_out, v_mid, counts, &eng1)) != TAC_OK)
    return st;
  if ((st = validate_call(&last, prep2, in2, real, v_mid, out2, v_final, counts ? cnt2 : nullptr, &eng2)) !=
      TAC_OK)
    return st;
  if ((st = launch_call(&full, gf, eng1, prepared, plan_exp(plan, 0), input, real, v_init, spikes_out, v_mid, counts, stream,
                        &launches)) != TAC_OK)
    return st;
  if ((st = launch_call(&last, gl, eng2, prep2, plan_exp(plan, 1), in2, real, v_mid, out2, v_final, counts ? cnt2 : nullptr,
                        stream, &launches)) != TAC_OK)
    return st;
  if (counts) {
    const int e = tacsnn::launch_add_u32(counts, cnt2, (long long)desc->B * desc->C_out, stream);
    if (e) return fail(TAC_ERR_CUDA, "count merge: %s", cudaGetErrorString((cudaError_t)e));
    ++launches;
  }
  g_launches = launches;
  return TAC_OK;
}
}  // namespace

extern "C" {

tac_status tac_conv_lif_forward(const tac_conv_lif_desc *desc, const tac_plan *plan,
                                const uint32_t *spikes_in, const float *v_init,
                                uint32_t *spikes_out, float *v_final, uint32_t *counts,
                                void *ws, size_t ws_bytes, void *stream) {
  return forward_impl(desc, plan, spikes_in, false, v_init, spikes_out, v_final, counts, ws, ws_bytes,
                      stream);
}

tac_status tac_conv_lif_forward_real(const tac_conv_lif_desc *desc, const tac_plan *plan,
                                     const float *x_in, const float *v_init,
                                     uint32_t *spikes_out, float *v_final, uint32_t *counts,
                                     void *ws, size_t ws_bytes, void *stream) {
  return forward_impl(desc, plan, x_in, true, v_init, spikes_out, v_final, counts, ws, ws_bytes,
                      stream);
}

}  // extern "C"

namespace {
// shared checks of the training calls: plan, no split call, subtract reset, unpooled output,
// at most kMaxTrainSteps LIF steps
constexpr int kMaxTrainSteps = 64;
tac_status train_checks(const tac_conv_lif_desc *desc, const tac_plan *plan, Geo *g) {
  tac_status st = check(desc, g);
  if (st != TAC_OK) return st;
  if (!plan) return fail(TAC_ERR_NULL, "plan is NULL");
  if (plan->abi_version != TACSNN_ABI_VERSION) return fail(TAC_ERR_PARAM, "plan from another ABI version");
  if (is_split_call(desc, *g))
    return fail(TAC_ERR_UNSUPPORTED, "training calls need K | T (no partial last group)");
  if (plan->fingerprint != fingerprint(desc, *g, false))
    return fail(TAC_ERR_PARAM, "plan was prepared for a different descriptor (see tac_plan)");
  if (plan->bytes < prep_total(desc, *g)) return fail(TAC_ERR_WORKSPACE, "plan image too small");
  if (desc->reset != TAC_RESET_SUBTRACT)
    return fail(TAC_ERR_UNSUPPORTED, "training calls support the subtract reset (PAPER.md:587-588)");
  if (desc->out_pool != 1)
    return fail(TAC_ERR_UNSUPPORTED, "training calls need out_pool = 1 (pool with tac_or_pool2)");
  if (g->G * g->nsteps > kMaxTrainSteps)
    return fail(TAC_ERR_UNSUPPORTED, "training calls support at most %d LIF steps", kMaxTrainSteps);
  return TAC_OK;
}
}  // namespace

extern "C" {

tac_status tac_conv_lif_forward_train(const tac_conv_lif_desc *desc, const tac_plan *plan, const void *input,
                                      const float *v_init, uint32_t *spikes_out, float *v_final,
                                      uint32_t *counts, float *y_seq, void *stream) {
  g_detail.clear();
  g_launches = 0;
  Geo g;
  tac_status st = train_checks(desc, plan, &g);
  if (st != TAC_OK) return st;
  if (!y_seq) return fail(TAC_ERR_NULL, "y_seq is NULL");
  if ((uintptr_t)y_seq % 4) return fail(TAC_ERR_ALIGN, "y_seq misaligned");
  if (!is_device_ptr(y_seq)) return fail(TAC_ERR_PARAM, "y_seq is not device memory");
  const bool real = desc->input_kind == TAC_INPUT_REAL;
  int engine;
  st = validate_call(desc, plan->prepared, input, real, v_init, spikes_out, v_final, counts, &engine);
  if (st != TAC_OK) return st;
  int launches = 0;
  st = launch_call(desc, g, engine, plan->prepared, plan_exp(plan, 0), input, real, v_init, spikes_out, v_final, counts, stream,
                   &launches, y_seq);
  if (st == TAC_OK) g_launches = launches;
  return st;
}

// the tcgen05 input gradient's weight image (bwd_tc.cu) follows dL/dY in the backward
// workspace for the shapes it takes (a layer whose forward runs on tcgen05)
// ... and the weight gradient's bf16 A_k buffer (tcgen05 layers with C_out >= 64)
size_t bwd_wgrad_abuf_bytes(const tac_conv_lif_desc *d, const Geo &g) {
  const bool ok = resolve_engine(d) == TAC_ENGINE_TCGEN05 && d->R == 3 && d->S == 3 && d->stride == 1 &&
                  (d->pad == 0 || d->pad == 1) && d->input_kind == TAC_INPUT_SPIKES &&
                  (d->C_in <= 8 || (d->C_in % 16 == 0 && d->C_in <= 128)) && d->C_out >= 64 && d->C_out <= 128 &&
                  d->C_out % 8 == 0;
  return ok ? align256(tacsnn::wgrad_tc_ws_bytes(g.G, d->B, d->H, d->W, d->C_in, g.Ho, g.Wo, d->C_out)) : 0;
}

// ... and, for a fully connected layer, the aggregated input and its gradient (GEMM path)
size_t bwd_fc_bytes(const tac_conv_lif_desc *d, const Geo &g) {
  const bool fc = d->H == 1 && d->W == 1 && d->R == 1 && d->S == 1 && d->pad == 0 && d->stride == 1;
  return fc ? 2 * align256((size_t)g.G * d->B * d->C_in * 4) : 0;
}

size_t bwd_dgrad_img_bytes(const tac_conv_lif_desc *d) {
  const bool ok = resolve_engine(d) == TAC_ENGINE_TCGEN05 && d->R == 3 && d->S == 3 && d->stride == 1 &&
                  (d->pad == 0 || d->pad == 1) && (d->C_in == 32 || d->C_in == 64 || d->C_in == 128) &&
                  d->C_out % 32 == 0;
  return ok ? align256(tacsnn::dgrad_tc_ws_bytes(d->C_in, d->C_out)) : 0;
}

tac_status tac_backward_workspace_bytes(const tac_conv_lif_desc *desc, size_t *bytes) {
  g_detail.clear();
  Geo g;
  tac_status st = check(desc, &g);
  if (st != TAC_OK) return st;
  if (!bytes) return fail(TAC_ERR_NULL, "bytes is NULL");
  *bytes = align256((size_t)g.G * desc->B * g.Ho * g.Wo * desc->C_out * 4) + bwd_dgrad_img_bytes(desc) +
           bwd_wgrad_abuf_bytes(desc, g) + bwd_fc_bytes(desc, g);
  return TAC_OK;
}

tac_status tac_conv_lif_backward(const tac_conv_lif_desc *desc, const tac_plan *plan,
                                 const tac_grad_desc *grad, const void *input, const float *v_init,
                                 const float *y_seq, const float *g_spikes, const float *g_v_final,
                                 float *g_weight, float *g_bias, float *g_input, float *g_v_init,
                                 float *g_agg_weights, void *ws, size_t ws_bytes, void *stream) {
  g_detail.clear();
  g_launches = 0;
  Geo g;
  tac_status st = train_checks(desc, plan, &g);
  if (st != TAC_OK) return st;
  if (!grad) return fail(TAC_ERR_NULL, "grad is NULL");
  if (grad->surrogate != TAC_SURROGATE_FAST_SIGMOID && grad->surrogate != TAC_SURROGATE_ARCTAN)
    return fail(TAC_ERR_PARAM, "surrogate=%d not in {0,1}", grad->surrogate);
  if (!std::isfinite(grad->alpha) || !(grad->alpha > 0.f))
    return fail(TAC_ERR_PARAM, "surrogate alpha must be finite and > 0");
  if (grad->detach_reset != 0 && grad->detach_reset != 1) return fail(TAC_ERR_PARAM, "detach_reset not in {0,1}");
  if (!input || !y_seq || !g_spikes || !g_weight || !g_bias) return fail(TAC_ERR_NULL, "NULL buffer");
  size_t need = 0;
  tac_backward_workspace_bytes(desc, &need);
  if (!ws) return fail(TAC_ERR_NULL, "workspace is NULL");
  if (ws_bytes < need) return fail(TAC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  const bool real = desc->input_kind == TAC_INPUT_REAL;
  const void *ptrs[] = {input, v_init, y_seq, g_spikes, g_v_final, g_weight, g_bias, g_input, g_v_init,
                        g_agg_weights, ws};
  const char *names[] = {"input", "v_init", "y_seq", "g_spikes", "g_v_final", "g_weight", "g_bias", "g_input",
                         "g_v_init", "g_agg_weights", "ws"};
  for (int i = 0; i < 11; ++i) {
    if (ptrs[i] && (uintptr_t)ptrs[i] % 4) return fail(TAC_ERR_ALIGN, "%s misaligned", names[i]);
    if (ptrs[i] && !is_device_ptr(ptrs[i])) return fail(TAC_ERR_PARAM, "%s is not device memory", names[i]);
  }
  const int engine = resolve_engine(desc);
  if (engine < 0) return fail(TAC_ERR_UNSUPPORTED, "engine TCGEN05 cannot run this layer");
  const PrepLayout L = prep_layout(desc);
  const unsigned char *base = static_cast<const unsigned char *>(plan->prepared);
  tacsnn::BwdParams p{};
  p.T = desc->T; p.B = desc->B; p.Cin = desc->C_in; p.H = desc->H; p.W = desc->W; p.Cout = desc->C_out;
  p.R = desc->R; p.S = desc->S; p.stride = desc->stride; p.pad = desc->pad; p.K = g.K; p.mode = desc->mode;
  p.G = g.G; p.nsteps = g.nsteps; p.Ho = g.Ho; p.Wo = g.Wo; p.wpr_in = g.wpr_in;
  p.in_st = g.in_st; p.in_sb = g.in_sb;
  const double beta = (double)desc->beta;
  p.decay = (float)(desc->mode == TAC_MODE_TAC ? std::pow(beta, (double)g.K) : beta);  // as the forward
  p.v_th = desc->v_th;
  const bool alpha = desc->agg_weights && desc->mode != TAC_MODE_DENSE;
  for (int j = 0; j < g.K; ++j)
    p.coef[j] = alpha ? desc->agg_weights[j] : (float)std::pow(beta, (double)(g.K - 1 - j));
  p.udomain = engine == TAC_ENGINE_TCGEN05 && tacsnn::tc_u_domain(desc);
  p.yscale = engine == TAC_ENGINE_TCGEN05 ? tacsnn::tc_yscale_ptr(desc, base + L.tc_off) : nullptr;
  p.surrogate = grad->surrogate;
  p.detach = grad->detach_reset;
  p.sg_alpha = grad->alpha;
  p.in = real ? nullptr : static_cast<const uint32_t *>(input);
  p.xin = real ? static_cast<const float *>(input) : nullptr;
  p.v_init = v_init; p.y_seq = y_seq; p.g_spikes = g_spikes; p.g_vfinal = g_v_final;
  p.g_y = static_cast<float *>(ws); p.g_vinit = g_v_init;
  const size_t gy_bytes = align256((size_t)g.G * desc->B * g.Ho * g.Wo * desc->C_out * 4);
  p.dg_img = bwd_dgrad_img_bytes(desc) ? static_cast<unsigned char *>(ws) + gy_bytes : nullptr;
  p.tc = engine == TAC_ENGINE_TCGEN05 ? 1 : 0;
  p.wg_abuf = bwd_wgrad_abuf_bytes(desc, g) ? static_cast<unsigned char *>(ws) + gy_bytes + bwd_dgrad_img_bytes(desc)
                                            : nullptr;
  p.fc_ws = bwd_fc_bytes(desc, g) ? static_cast<unsigned char *>(ws) + gy_bytes + bwd_dgrad_img_bytes(desc) +
                                        bwd_wgrad_abuf_bytes(desc, g)
                                  : nullptr;
  p.w = reinterpret_cast<const float *>(base + L.simt_off);
  p.g_w = g_weight; p.g_b = g_bias; p.g_in = g_input; p.g_alpha = g_agg_weights;
  int launches = 0;
  const int e = tacsnn::launch_backward(p, stream, &launches);
  if (e) return fail(TAC_ERR_CUDA, "backward launch: %s", cudaGetErrorString((cudaError_t)e));
  g_launches = launches;
  return TAC_OK;
}

tac_status tac_or_pool2(const uint32_t *in, uint32_t *out, int32_t T, int32_t B, int32_t C, int32_t H,
                        int32_t W, void *stream) {
  g_detail.clear();
  if (!in || !out) return fail(TAC_ERR_NULL, "NULL buffer");
  if (T < 1 || B < 1 || C < 1 || H < 2 || W < 2) return fail(TAC_ERR_SHAPE, "extent < 1 (H, W >= 2)");
  if ((uintptr_t)in % 4 || (uintptr_t)out % 4) return fail(TAC_ERR_ALIGN, "misaligned");
  const int e = tacsnn::launch_or_pool2(in, out, T, B, C, H, W, stream);
  if (e) return fail(TAC_ERR_CUDA, "or_pool2: %s", cudaGetErrorString((cudaError_t)e));
  g_launches = 1;
  return TAC_OK;
}

tac_status tac_or_pool2_backward(const uint32_t *spikes_prepool, const float *g_pooled, float *g_prepool,
                                 int32_t T, int32_t B, int32_t C, int32_t H, int32_t W, void *stream) {
  g_detail.clear();
  if (!spikes_prepool || !g_pooled || !g_prepool) return fail(TAC_ERR_NULL, "NULL buffer");
  if (T < 1 || B < 1 || C < 1 || H < 2 || W < 2) return fail(TAC_ERR_SHAPE, "extent < 1 (H, W >= 2)");
  if ((uintptr_t)spikes_prepool % 4 || (uintptr_t)g_pooled % 4 || (uintptr_t)g_prepool % 4)
    return fail(TAC_ERR_ALIGN, "misaligned");
  const int e = tacsnn::launch_or_pool2_backward(spikes_prepool, g_pooled, g_prepool, T, B, C, H, W, stream);
  if (e) return fail(TAC_ERR_CUDA, "or_pool2_backward: %s", cudaGetErrorString((cudaError_t)e));
  g_launches = 1;
  return TAC_OK;
}

tac_status tac_vote(const uint32_t *counts, int32_t B, int32_t C, int32_t voters, int32_t T_out,
                    float *scores, void *stream) {
  g_detail.clear();
  if (!counts || !scores) return fail(TAC_ERR_NULL, "NULL buffer");
  if (B < 1 || C < 1 || voters < 1 || T_out < 1 || C % voters)
    return fail(TAC_ERR_SHAPE, "need B, C, voters, T_out >= 1 and C %% voters == 0");
  if ((uintptr_t)counts % 4 || (uintptr_t)scores % 4) return fail(TAC_ERR_ALIGN, "misaligned");
  const int e = tacsnn::launch_vote(counts, B, C, voters, T_out, scores, stream);
  if (e) return fail(TAC_ERR_CUDA, "vote: %s", cudaGetErrorString((cudaError_t)e));
  g_launches = 1;
  return TAC_OK;
}

tac_status tac_pack_spikes(const uint8_t *dense01, uint32_t *packed, int32_t T, int32_t B,
                           int32_t C, int32_t H, int32_t W, void *stream) {
  g_detail.clear();
  if (!dense01 || !packed) return fail(TAC_ERR_NULL, "NULL buffer");
  if (T < 1 || B < 1 || C < 1 || H < 1 || W < 1) return fail(TAC_ERR_SHAPE, "extent < 1");
  if ((uintptr_t)packed % 4) return fail(TAC_ERR_ALIGN, "packed misaligned");
  int e = tacsnn::launch_pack(dense01, packed, T, B, C, H, W, stream);
  if (e) return fail(TAC_ERR_CUDA, "pack: %s", cudaGetErrorString((cudaError_t)e));
  g_launches = 1;
  return TAC_OK;
}

tac_status tac_unpack_spikes(const uint32_t *packed, uint8_t *dense01, int32_t T, int32_t B,
                             int32_t C, int32_t H, int32_t W, void *stream) {
  g_detail.clear();
  if (!dense01 || !packed) return fail(TAC_ERR_NULL, "NULL buffer");
  if (T < 1 || B < 1 || C < 1 || H < 1 || W < 1) return fail(TAC_ERR_SHAPE, "extent < 1");
  if ((uintptr_t)packed % 4) return fail(TAC_ERR_ALIGN, "packed misaligned");
  int e = tacsnn::launch_unpack(packed, dense01, T, B, C, H, W, stream);
  if (e) return fail(TAC_ERR_CUDA, "unpack: %s", cudaGetErrorString((cudaError_t)e));
  g_launches = 1;
  return TAC_OK;
}

const char *tac_status_string(tac_status s) {
  switch (s) {
    case TAC_OK: return "TAC_OK";
    case TAC_ERR_NULL: return "TAC_ERR_NULL";
    case TAC_ERR_SHAPE: return "TAC_ERR_SHAPE";
    case TAC_ERR_K_NOT_DIVIDING_T: return "TAC_ERR_K_NOT_DIVIDING_T";
    case TAC_ERR_PARAM: return "TAC_ERR_PARAM";
    case TAC_ERR_NONFINITE: return "TAC_ERR_NONFINITE";
    case TAC_ERR_ALIGN: return "TAC_ERR_ALIGN";
    case TAC_ERR_UNSUPPORTED: return "TAC_ERR_UNSUPPORTED";
    case TAC_ERR_WORKSPACE: return "TAC_ERR_WORKSPACE";
    case TAC_ERR_CUDA: return "TAC_ERR_CUDA";
  }
  return "TAC_ERR_UNKNOWN";
}

const char *tac_last_error_detail(void) { return g_detail.c_str(); }
int32_t tac_abi_version(void) { return TACSNN_ABI_VERSION; }
int32_t tac_last_launch_count(void) { return g_launches; }

}  // extern "C"
