// tc.cu -- host side of the tcgen05 engine of libtacsnn: weight preparation (the
// resident SMEM image of each CTA of the pair), the tensor maps, the kernel
// parameters and the launch.  The fused kernel itself (aggregation + tcgen05 conv +
// LIF epilogue) is in tc_impl.cuh and instantiated by tc_k_*.cu.
#include "tc_impl.cuh"

namespace tacsnn {
namespace {

__global__ void tc_zero_kernel(uint32_t *out, int T_out, int B, long long plane, long long st,
                               long long sb, uint32_t *counts, long long ncounts) {
  const long long total = (long long)T_out * B * plane;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long tb = i / plane, o = i - tb * plane;
    const long long t = tb / B, b = tb - t * B;
    out[t * st + b * sb + o] = 0u;
  }
  if (counts)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ncounts; i += stride)
      counts[i] = 0u;
}


}  // namespace

// ------------------------------------------------------------------ host API --
static bool lif_u_state(const tac_conv_lif_desc *d);
bool tc_u_domain(const tac_conv_lif_desc *d) { return !fc_is_fc(d) && lif_u_state(d); }
bool tc_shape_ok(const tac_conv_lif_desc *d) {
  return fc_is_fc(d) ? fc_reason(d) == nullptr : shape_reason(d) == nullptr;
}
bool tc_supported(const tac_conv_lif_desc *d) { return fc_is_fc(d) ? fc_reason(d) == nullptr : reason(d) == nullptr; }
const char *tc_unsupported_reason(const tac_conv_lif_desc *d) {
  const char *r = fc_is_fc(d) ? fc_reason(d) : reason(d);
  return r ? r : "supported";
}

// The specialised subtract-reset epilogue (NS > 0) integrates U = decay V + Y'' with the
// drive Y'' = Y - v_th: the offset is folded into the prepared bias.
static bool lif_u_state(const tac_conv_lif_desc *d) {
  const int ns = d->mode == TAC_MODE_TACTP ? d->K : 1;
  return d->reset == TAC_RESET_SUBTRACT && (ns == 1 || ns == 2 || ns == 4 || ns == 8);
}
static double lif_bias_offset(const tac_conv_lif_desc *d) {
  return lif_u_state(d) ? -(double)d->v_th : 0.0;
}

// Image: [slice 0 | slice 1 | fp32 [s1/254 | bias | s1 | s2] x C_out_pad | fp32 yscale [4] |
//         u32 aggregate tables [kLutWords] (split path only)]
static size_t scale_off(const Geometry &g) { return 2 * (size_t)g.w_bytes_cta; }
static size_t yscale_off(const Geometry &g) { return scale_off(g) + 16 * (size_t)g.cout_pad; }
static size_t lut_off(const Geometry &g) { return yscale_off(g) + 16; }
size_t tc_weights_bytes(const tac_conv_lif_desc *d) {
  if (fc_is_fc(d)) return fc_weights_bytes(d);
  const Geometry g = geometry(d);
  return lut_off(g) + (g.split ? 4 * (size_t)kLutWords : 0);
}
const float *tc_yscale_ptr(const tac_conv_lif_desc *d, const unsigned char *tc_prep) {
  if (fc_is_fc(d)) return nullptr;  // the FC epilogue hands the LIF the unscaled Y (V domain)
  const Geometry g = geometry(d);
  return g.path == PATH_HALO ? nullptr : reinterpret_cast<const float *>(tc_prep + yscale_off(g));
}

// Two int8 slices per output channel, laid out as the smem image of each CTA:
// halo  : [tap][kc16][n][16 B], K index 32w + 4o + b <-> channel 32w + o + 8b
// h16   : fp16 hi/lo slices over a 16-channel halo pixel, see below
// followed by fp32 [s1/254 | bias | s1 | s2] per padded output channel.
int tc_prepare(const tac_conv_lif_desc *d, const float *weight, const float *bias,
               unsigned char *dst) {
  if (fc_is_fc(d)) return fc_prepare(d, weight, dst);
  const Geometry g = geometry(d);
  const int Co = d->C_out, Ci = d->C_in, Cp = g.cout_pad;
  std::vector<signed char> q1((size_t)Cp * Ci * 9, 0), q2((size_t)Cp * Ci * 9, 0);
  std::vector<float> s1(Cp, 0.f), s2(Cp, 0.f), bs(Cp, 0.f);
  const double boff = lif_bias_offset(d);
  for (int co = 0; co < Co; ++co) {
    bs[co] = (float)((bias ? (double)bias[co] : 0.0) + boff);
    double amax = 0.0;
    for (int i = 0; i < Ci * 9; ++i) amax = std::max(amax, std::fabs((double)weight[(size_t)co * Ci * 9 + i]));
    if (amax == 0.0) continue;
    s1[co] = (float)(amax / 127.0);
    const double sc1 = (double)s1[co], sc2 = sc1 / 254.0;  // lo slice step = s1 / 254
    s2[co] = (float)sc2;
    for (int i = 0; i < Ci * 9; ++i) {
      const double w = weight[(size_t)co * Ci * 9 + i];
      const double a = std::max(-127.0, std::min(127.0, std::nearbyint(w / sc1)));
      const double r = w - a * sc1;
      const double b = std::max(-127.0, std::min(127.0, std::nearbyint(r / sc2)));
      q1[(size_t)co * Ci * 9 + i] = (signed char)a;
      q2[(size_t)co * Ci * 9 + i] = (signed char)b;
    }
  }
  auto q_at = [&](int half, int co, int ci, int r, int s) -> signed char {
    const std::vector<signed char> &q = half ? q2 : q1;
    return q[(((size_t)co * Ci + ci) * 3 + r) * 3 + s];
  };
  double ysc = 1.0;  // fp16 paths: 2^e (see below); int8 path: 1
  int yexp = 0;
  if (g.path != PATH_HALO) {
    const int m = (d->mode == TAC_MODE_DENSE || g.split) ? 0 : beta_shift(d->beta);
    const int Kg = d->mode == TAC_MODE_DENSE ? 1 : d->K;
    const double agg = g.split ? 1.0 : std::ldexp(1.0, -m * (Kg - 1));
    double mx = 0.0;
    for (int co = 0; co < Co; ++co) {
      for (int i = 0; i < Ci * 9; ++i) mx = std::max(mx, std::fabs((double)weight[(size_t)co * Ci * 9 + i]) * agg);
      mx = std::max(mx, std::fabs((bias ? (double)bias[co] : 0.0) + boff));
    }
    if (mx > 0.0) yexp = std::max(-60, std::min(60, -std::ilogb(mx)));
    ysc = std::ldexp(1.0, yexp);
  }
  for (int half = 0; half < 2; ++half) {
    unsigned char *img = dst + (size_t)half * g.w_bytes_cta;
    std::memset(img, 0, g.w_bytes_cta);
    if (g.path == PATH_HALO) {
      for (int tap = 0; tap < 9; ++tap)
        for (int kidx = 0; kidx < Ci; ++kidx) {
          const int w32 = kidx / 32, o = (kidx % 32) / 4, b = kidx % 4;
          const int ci = 32 * w32 + o + 8 * b;
          const int kc = kidx / 16, byte = kidx % 16;
          for (int n = 0; n < Cp; ++n)
            img[(((size_t)tap * g.nkc + kc) * Cp + n) * 16 + byte] =
                (unsigned char)(n < Co ? q_at(half, n, ci, tap / 3, tap % 3) : 0);
        }
    } else {
      // fp16 image, CTA `half` holds output channels [half*Cp/2, (half+1)*Cp/2) of BOTH
      // slices: [slice][tap][16-B chunk (nkc)][row (Cp/2)][8 fp16].  Halo channel k:
      //   exact u8 aggregate : k < C_in -> W[n][k][r][s] * 2^{-m(K-1)} (folded scale),
      //                        k == C_in of the centre tap -> bias (producers store 1.0)
      //   split A (hi | lo)  : k < C_in -> W (hi slice: fp16 hi, lo slice: fp16 lo),
      //                        C_in <= k < 2 C_in -> W hi in the hi slice (times A_lo),
      //                        0 in the lo slice (A_lo W_lo ~ 2^-33 |A W|), bias at 2 C_in
      // so D = sum (A_hi + A_lo) W_hi + A_hi W_lo + bias, accumulated in fp32.
      const bool split = g.split != 0;
      const int m = (d->mode == TAC_MODE_DENSE || split) ? 0 : beta_shift(d->beta);
      const int Kg = d->mode == TAC_MODE_DENSE ? 1 : d->K;
      // layer prescale 2^e: the largest operand |w agg| or |bias + offset| lands in [1, 2),
      // so the fp16 hi + lo pair keeps ~22 bits of every value relative to the layer's
      // scale (no absolute 2^-24 quantum, no overflow past 65504); the epilogue runs the
      // LIF in the same scale (yscale)
      const double agg = (split ? 1.0 : std::ldexp(1.0, -m * (Kg - 1))) * ysc;
      const int nh = Cp / 2, nk = g.nkc, kbias = split ? 2 * Ci : Ci;
      uint16_t *img16 = reinterpret_cast<uint16_t *>(img);
      if (packed_of(d)) {
        // packed slices (one MMA per tap): slice 0 holds [W_hi | b_hi | W_lo | b_lo] against
        // the halo channels [A | 1 | A | 1]; slice 1 stays zero (not read)
        for (int nl = 0; nl < nh; ++nl) {
          const int n = half * nh + nl;
          for (int tap = 0; tap < 9; ++tap)
            for (int k = 0; k < 8 * nk; ++k) {
              // exact: [W (C_in) | b] hi then lo; split: [W (C_in) | W (C_in) | b] hi then [W | b] lo
              const int nhi = split ? 2 * Ci + 1 : Ci + 1;
              const int part = k < nhi ? 0 : (k < nhi + Ci + 1 ? 1 : 2);  // 0: hi, 1: lo, 2: pad
              const int kk = part == 0 ? k : k - nhi;
              const int nw = part == 0 && split ? 2 * Ci : Ci;  // weight channels before the bias
              double wv = 0.0;
              if (n < Co && part < 2) {
                if (kk < nw) wv = (double)weight[(((size_t)n * Ci + kk % Ci) * 3 + tap / 3) * 3 + tap % 3] * agg;
                else if (kk == nw && tap == 4) wv = ((bias ? (double)bias[n] : 0.0) + boff) * ysc;
              }
              const __half hi = __double2half(wv);
              const __half v = part == 0 ? hi : __double2half(part == 1 ? wv - (double)__half2float(hi) : 0.0);
              img16[((((size_t)0 * 9 + tap) * nk + k / 8) * nh + nl) * 8 + k % 8] = __half_as_ushort(v);
            }
        }
        continue;
      }
      for (int nl = 0; nl < nh; ++nl) {
        const int n = half * nh + nl;
        for (int tap = 0; tap < 9; ++tap)
          for (int k = 0; k < 8 * nk; ++k) {
            double wv = 0.0;
            bool hi_only = false;
            if (n < Co) {
              const int ci = k < Ci ? k : (split && k < 2 * Ci ? k - Ci : -1);
              if (ci >= 0) {
                wv = (double)weight[(((size_t)n * Ci + ci) * 3 + tap / 3) * 3 + tap % 3] * agg;
                hi_only = k >= Ci;
              } else if (k == kbias && tap == 4) {
                wv = ((bias ? (double)bias[n] : 0.0) + boff) * ysc;
              }
            }
            const __half hi = __double2half(wv);
            const __half lo = hi_only ? __double2half(0.0) : __double2half(wv - (double)__half2float(hi));
            const int ck = k / 8, e = k % 8;
            img16[((((size_t)0 * 9 + tap) * nk + ck) * nh + nl) * 8 + e] = __half_as_ushort(hi);
            img16[((((size_t)1 * 9 + tap) * nk + ck) * nh + nl) * 8 + e] = __half_as_ushort(lo);
          }
      }
    }
  }
  // [s1/254 | bias | s1 | s2] (the kernel multiplies all but bias by 2^{-m(K-1)})
  float *sb = reinterpret_cast<float *>(dst + scale_off(g));
  for (int i = 0; i < Cp; ++i) {
    sb[i] = (float)((double)s1[i] / 254.0);
    sb[Cp + i] = bs[i];
    sb[2 * Cp + i] = s1[i];
    sb[3 * Cp + i] = s2[i];
  }
  float *ys = reinterpret_cast<float *>(dst + yscale_off(g));
  ys[0] = (float)ysc;
  ys[1] = (float)(1.0 / ysc);
  ys[2] = ys[3] = 0.f;
  if (g.split) {
    // aggregate tables (split path): A = sum_j c_j bit_j with c_j = alpha_j (learnable,
    // PAPER.md:427) or beta^{K-1-j} (Definition TAC), built in fp64
    uint32_t *lut = reinterpret_cast<uint32_t *>(dst + lut_off(g));
    std::memset(lut, 0, 4 * (size_t)kLutWords);
    const int K = d->mode == TAC_MODE_DENSE ? 1 : d->K;
    std::vector<double> c(K);
    for (int j = 0; j < K; ++j)
      c[j] = d->agg_weights ? (double)d->agg_weights[j] : std::pow((double)d->beta, (double)(K - 1 - j));
    auto sum_bits = [&](int idx, int j0, int n) {
      double a = 0.0;
      for (int j = 0; j < n; ++j)
        if ((idx >> j) & 1) a += c[j0 + j];
      return a;
    };
    if (K <= 8) {
      for (int idx = 0; idx < 256; ++idx) {
        const double a = sum_bits(idx, 0, K);
        const __half hi = __double2half(a);
        const __half lo = __double2half(a - (double)__half2float(hi));
        lut[idx] = (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
      }
    } else {  // two fp32 half tables: frames 0..K-9 and K-8..K-1
      const int ka = K - 8;
      for (int idx = 0; idx < 256; ++idx) {
        const float fa = (float)sum_bits(idx, 0, ka), fb = (float)sum_bits(idx, ka, 8);
        std::memcpy(&lut[256 + idx], &fa, 4);
        std::memcpy(&lut[512 + idx], &fb, 4);
      }
    }
  }
  return yexp;
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    else
      cudaGetLastError();
  }
  return fn;
}
}  // namespace

// Debug timeline (not part of the ABI contract): when tac_debug_set_trace() was
// given a device buffer of >= 4096 * 8 u64, CTA 0 of every tcgen05 launch records
// %globaltimer per group iteration and role event (see TR_* slots).
static unsigned long long *g_trace = nullptr;
unsigned long long *tacsnn_trace_buffer() { return g_trace; }
extern "C" void tac_debug_set_trace(void *dev) {
  g_trace = reinterpret_cast<unsigned long long *>(dev);
}

int tc_launch(const tac_conv_lif_desc *d, const LayerParams &lp, const unsigned char *tc_prep,
              void *stream, int *launches) {
  if (fc_is_fc(d)) return fc_launch(d, lp, tc_prep, stream, launches);
  // TMA raw-halo producer when the packed input is a legal 4-D tensor-map view
  // (16-B aligned base and strides) and the plan fits in shared memory
  static const bool no_tma = [] { const char *e = std::getenv("TACSNN_NO_TMA"); return e && *e == '1'; }();
  const bool tma_layout = !no_tma && !lp.xin && (lp.wpr_in * 4) % 16 == 0 && (lp.in_sb * 4) % 16 == 0 &&
                          (lp.in_st * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(lp.in) % 16) == 0;
  // plane mode: narrow first-layer frames (e.g. 28 x 28 x 1 = 28 words = 112 B) whose row
  // stride is below TMA's 16-B granularity but whose whole frame is a legal box: one
  // 3-D box [K frames][H * WPR words] per group replaces per-pixel global loads
  const int plane = lp.H * lp.wpr_in;
  static const bool no_plane = [] { const char *e = std::getenv("TACSNN_NO_PLANE"); return e && *e == '1'; }();
  const bool plane_layout = !no_tma && !no_plane && !tma_layout && !lp.xin && lp.Cin <= 8 && plane <= 256 &&
                            (plane * 4) % 16 == 0 && (lp.in_sb * 4) % 16 == 0 && (lp.in_st * 4) % 16 == 0 &&
                            (reinterpret_cast<uintptr_t>(lp.in) % 16) == 0;
  Geometry g = plane_layout ? geometry(d, true, plane) : geometry(d, tma_layout);
  PFN_cuTensorMapEncodeTiled_v12000 encode = g.use_tma ? tensor_map_encoder() : nullptr;
  if (!encode) g = geometry(d, false);
  TcParams p{};
  if (g.use_tma && plane_layout) {
    const cuuint64_t dims[3] = {(cuuint64_t)plane, (cuuint64_t)lp.B, (cuuint64_t)lp.T};
    const cuuint64_t strides[2] = {(cuuint64_t)lp.in_sb * 4, (cuuint64_t)lp.in_st * 4};
    const cuuint32_t box[3] = {(cuuint32_t)plane, 1u, (cuuint32_t)lp.K};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void *)lp.in, dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) g = geometry(d, false);
  } else if (g.use_tma) {
    const int K = lp.K;
    const cuuint64_t dims[4] = {(cuuint64_t)lp.wpr_in, (cuuint64_t)lp.H, (cuuint64_t)lp.B,
                                (cuuint64_t)lp.T};
    const cuuint64_t strides[3] = {(cuuint64_t)lp.wpr_in * 4, (cuuint64_t)lp.in_sb * 4,
                                   (cuuint64_t)lp.in_st * 4};
    const cuuint32_t box[4] = {(cuuint32_t)g.raw_bw, (cuuint32_t)kHaloH, 1u, (cuuint32_t)K};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, (void *)lp.in, dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) g = geometry(d, false);
  }
  p.use_tma = g.use_tma ? (plane_layout ? 2 : 1) : 0;
  // first layers with pixel-wise producers (LDG or whole-plane TMA): a producer warp per A
  // stage, so three stages are built concurrently (one stage's latency -- loads, table
  // lookups, the async-proxy fence -- no longer serialises the pipeline)
  static const bool no_ws = [] { const char *e = std::getenv("TACSNN_NO_WARP_STAGE"); return e && *e == '1'; }();
  static const bool no_hrows = [] { const char *e = std::getenv("TACSNN_NO_HALO_ROWS"); return e && *e == '1'; }();
  p.warp_stage = (!no_ws && g.path != PATH_HALO && (p.use_tma != 1 || (!no_hrows && rows_ok(d)))) ? 1 : 0;
  p.prod_step = p.warp_stage ? 32 : 32 * kProdWarps;
  static const bool no_pr = [] { const char *e = std::getenv("TACSNN_NO_PROD_REFILL"); return e && *e == '1'; }();
  p.prod_refill = (!no_pr && p.warp_stage && p.use_tma != 0) ? 1 : 0;
  p.raw_bw = g.raw_bw;
  p.nraw = g.nraw;
  p.off_raw = g.off_raw;
  p.raw_stage_bytes = g.raw_stage_bytes;
  p.raw_box_bytes = g.raw_box_bytes;
  p.B = lp.B; p.H = lp.H; p.W = lp.W; p.Cin = lp.Cin; p.Cout = lp.Cout; p.Cout_pad = g.cout_pad;
  p.pad = lp.pad; p.Ho = lp.Ho; p.Wo = lp.Wo; p.pool = lp.pool; p.Hq = lp.Hq; p.Wq = lp.Wq;
  p.K = lp.K; p.G = lp.G; p.nsteps = lp.nsteps; p.mode = lp.mode; p.reset = lp.reset;
  p.tiles_x = (lp.Wo + kTileW - 1) / kTileW;
  p.tiles_y = (lp.Ho + kTileH - 1) / kTileH;
  p.num_tiles = lp.B * p.tiles_x * p.tiles_y;
  p.num_pairs = (p.num_tiles + 1) / 2;
  p.nstages = g.nstages;
  p.nkc = g.nkc; p.ntaps = g.ntaps;
  p.m_shift = (d->mode == TAC_MODE_DENSE || g.split) ? 0 : beta_shift(d->beta);
  p.split = g.split;
  p.off_lut = g.off_lut;
  p.real = lp.xin ? 1 : 0;
  p.xin = lp.xin;
  for (int j = 0; j < 16; ++j) p.coef[j] = j < lp.K ? lp.coef[j] : 0.f;
  p.lut_g = reinterpret_cast<const uint32_t *>(tc_prep + lut_off(g));  // split: prepared tables
  p.ysc = (float)std::ldexp(1.0, g.path == PATH_HALO ? 0 : lp.yscale_exp);  // the plan's prescale
  p.iysc = (float)std::ldexp(1.0, g.path == PATH_HALO ? 0 : -lp.yscale_exp);
  p.vth_s = lp.v_th * p.ysc;
  p.wpr_in = lp.wpr_in; p.wpr_out = lp.wpr_out;
  p.nwo = lp.Cout % 32 == 0 ? lp.Cout / 32 : 1;
  static const bool no_c32w = [] { const char *e = std::getenv("TACSNN_NO_C32W"); return e && *e == '1'; }();
  p.c32w = (!no_c32w && g.path != PATH_HALO && g.cout_pad == 32) ? 1 : 0;
  // Waiting roles (measured per K on C5, scripts/gpu/ab_k.sh, A/B on one box): on the int8
  // (halo-path) layers with <= 4 LIF steps per group the producers, raw loader and MMA
  // issuer back off with nanosleep instead of suspend-hint waits that wake on every barrier
  // event (K=4: C5 L2 -2..-6 %, L3..L5 -3..-4 %; K=2 neutral), and with 4 steps the MMA
  // warp refills the raw slot after issuing (L3 / L4 -5 %).  With 8 steps per group both
  // lose (L2 +11 % / +41 %), as does any backoff on the fp16 first layers (+0.6..5 %).
  // A/B overrides: TACSNN_SLEEP_NS, TACSNN_REFILL_EARLY
  const bool halo_short = g.path == PATH_HALO && p.nsteps <= 4;
  static const int sleep_env = [] { const char *e = std::getenv("TACSNN_SLEEP_NS"); return e ? std::atoi(e) : -1; }();
  p.sleep_ns = sleep_env >= 0 ? sleep_env : (halo_short ? 512 : 0);
  static const int early_env = [] { const char *e = std::getenv("TACSNN_REFILL_EARLY"); return e ? std::atoi(e) : -1; }();
  p.refill_early = early_env >= 0 ? early_env : ((g.path == PATH_HALO && p.nsteps == 4) ? 0 : 1);
  const bool out_atomic = g.cout_pad < 64 && !p.c32w;  // sub-word or shared-word output fields
  {  // exact s32 combine 254 D_hi + D_lo possible? |A| <= A_max, |q| <= 127, K_red terms
    double a_max = 0;
    for (int j = 0; j < lp.K; ++j) a_max += std::ldexp(1.0, p.m_shift * j);
    const double kred = g.path == PATH_HALO ? 9.0 * lp.Cin : 32.0;
    p.int_combine = (a_max * 127.0 * kred * 255.0 < 2147483647.0) ? 1 : 0;
  }
  p.in_st = lp.in_st; p.in_sb = lp.in_sb; p.out_st = lp.out_st; p.out_sb = lp.out_sb;
  p.decay = lp.decay; p.v_th = lp.v_th; p.v_reset = lp.v_reset;
  p.agg_scale = (float)std::ldexp(1.0, -p.m_shift * (lp.K - 1));
  p.off_w = g.off_w; p.off_a = g.off_a; p.a_stage_bytes = g.a_stage_bytes;
  p.off_scale = g.off_scale; p.off_bar = g.off_bar;
  p.smem_bytes = g.smem_bytes; p.w_bytes_cta = g.w_bytes_cta;
  p.n_total = g.path == PATH_HALO ? 2u * g.cout_pad : (uint32_t)g.cout_pad;  // TMEM columns / acc
  uint32_t cols = 32;
  const bool ut = g.path != PATH_HALO && g.cout_pad == 128;  // u_in_tmem(): V after the accumulators
  // accumulators: 3 on the fp16 paths (n_total = C_out_pad; with V in TMEM 3 x 128 +
  // 128 = 512 columns), 2 on the int8 path (n_total = 2 C_out_pad)
  p.naccs = g.path == PATH_HALO ? 2 : TACSNN_H16_ACCS;
  if (p.warp_stage && g.cout_pad <= 64) p.naccs = kAccs;  // small first layers: deeper TMEM ring
  p.packed = packed_of(d) ? 1 : 0;
  while (cols < (uint32_t)p.naccs * p.n_total + (ut ? 128u : 0u)) cols <<= 1;
  p.tmem_cols = cols;
  p.lbo_a = (uint32_t)kHaloRows * 16u;  // between 16-byte K chunks
  p.sbo_a = (uint32_t)kHaloW * 16u;     // between tile rows (8-row core-matrix groups)
  for (int t = 0; t < 9; ++t) p.tap_off[t] = (t / 3) * kHaloW + (t % 3);
  // B: rows held by one CTA x 16 B between 16-byte K chunks
  p.lbo_b = g.path == PATH_HALO ? (uint32_t)g.cout_pad * 16u : (uint32_t)(g.cout_pad / 2) * 16u;
  p.in = lp.in; p.out = lp.out; p.v_init = lp.v_init; p.v_final = lp.v_final; p.counts = lp.counts;
  p.y_seq = lp.y_seq;
  p.yseq_plane = (long long)lp.B * lp.Ho * lp.Wo * lp.Cout;
  p.trace = tacsnn_trace_buffer();
  p.w_img = tc_prep;
  p.scale_bias = reinterpret_cast<const float *>(tc_prep + scale_off(g));

  cudaStream_t st = (cudaStream_t)stream;
  if (out_atomic || p.counts) {
    const long long plane = out_atomic ? (long long)lp.Hq * lp.wpr_out : 0;
    const long long total = std::max((long long)lp.T_out * lp.B * plane, (long long)lp.B * lp.Cout);
    const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    tc_zero_kernel<<<std::max(grid, 1), 256, 0, st>>>(p.out, lp.T_out, lp.B, plane, lp.out_st,
                                                       lp.out_sb, p.counts, (long long)lp.B * lp.Cout);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
  }
  // two pipelines per SM for the small first layers when their smem and TMEM halve
  static const bool no_occ2 = [] { const char *e = std::getenv("TACSNN_NO_OCC2"); return e && *e == '1'; }();
  p.occ = (!no_occ2 && p.warp_stage && g.path != PATH_HALO && g.cout_pad <= 32 && p.smem_bytes <= 112u * 1024u &&
           p.tmem_cols <= 256u) ? 2 : 1;
  const int nclusters = std::max(1, std::min(p.num_pairs, 74 * p.occ));
  const bool train = lp.y_seq != nullptr;
  cudaError_t e;
  if (g.path == PATH_HALO)
    e = train ? tc_launch_path<PATH_HALO, true>(p, g.cout_pad, nclusters, st)
              : tc_launch_path<PATH_HALO, false>(p, g.cout_pad, nclusters, st);
  else if (!g.split)
    e = train ? tc_launch_path<PATH_H16, true>(p, g.cout_pad, nclusters, st)
              : tc_launch_path<PATH_H16, false>(p, g.cout_pad, nclusters, st);
  else
    e = train ? tc_launch_path<PATH_SPLIT, true>(p, g.cout_pad, nclusters, st)
              : tc_launch_path<PATH_SPLIT, false>(p, g.cout_pad, nclusters, st);
  ++*launches;
  return (int)e;
}

}  // namespace tacsnn
