/*
 * tac_oracle.c -- plain, slow, obviously-correct CPU oracle for the Conv-LIF
 * layer of arXiv 2603.13810 (TAC / TAC-TP) and its per-timestep baseline.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2603_13810_b200/) never links, loads or calls it,
 * and this file shares no code, header, table or constant with that path.
 *
 * Precision: every value is fp64 (inputs are the fp32 weights / beta / v_th the
 * caller passes, promoted).  Layout is the paper's: spikes S in
 * {0,1}^{T x B x C x H x W}, time outermost (Alg. 1 "Require").
 *
 * Citations "P:n" are /root/reference/PAPER.md line n, "S:n" SPEC.md line n.
 *
 *   conv      : Y[b,co,y,x] = bias[co] + sum_{ci,r,s} W[co,ci,r,s] *
 *               X[b,ci,y*stride+r-pad, x*stride+s-pad]   (zero outside)
 *               -- cross-correlation with zero padding, S:51-55 (conv2d post);
 *               "W * S_t" of Eq. (1).
 *   dense     : Eq. (1): for t<T: V <- beta V + conv(S_t); spike; reset
 *   TAC       : Algorithm 1, P:135-150:
 *               A_k = sum_{j<K} beta^{K-1-j} S_{kK+j}      (Def. TAC)
 *               Y_k = Conv2d(A_k, W)                        (Alg.1 l.4)
 *               V <- beta^K V + Y_k ; S_k = Theta(V - V_th) ; V <- V - S_k V_th
 *   TAC-TP    : Algorithm 2: same A_k, Y_k; then K times
 *               V <- beta V + Y_k ; S_{kK+j} = Theta(V - V_th) ; V <- V - S V_th
 *
 * Readings:
 *   R1 reset: SUBTRACT is Alg.1/2 (immediate, then decayed); DELAYED is Eq. (1) /
 *      App. A (V_t = beta V_{t-1} + I_t - V_th S_{t-1}); HARD sets V = v_reset.
 *   R2 Theta(0) = 1: fire when V >= V_th ("fire at exact threshold").
 *   R3 bias added once per conv call (folded BN).
 *   R4 DELAYED at call start: s_prev = [v_init >= v_th] (0 when v_init = 0).
 *   R5 v_final = V after the last step (post-reset for SUBTRACT/HARD).
 *
 * Replay (parity protocol): when `replay` (device spikes, same
 * layout as `out`) is given, each threshold decision inside the band
 * |V - v_th| <= band takes the device spike (excused); outside it the oracle's
 * own decision is used and compared with the device spike (mismatch).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_MODE_DENSE = 0, OR_MODE_TAC = 1, OR_MODE_TACTP = 2 };
enum { OR_RESET_SUBTRACT = 0, OR_RESET_DELAYED = 1, OR_RESET_HARD = 2 };

int tac_oracle_abi(void) { return 1; }

int tac_oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of later calls (timing the single-core baseline). */
void tac_oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* Direct-loop 2-D cross-correlation of ONE sample.
 * X [Cin][H][W], Wt [Cout][Cin][R][S], bias [Cout] or NULL, Y [Cout][Ho][Wo]. */
static void conv_one(const double *X, const float *Wt, const float *bias,
                     int Cin, int H, int W, int Cout, int R, int S,
                     int stride, int pad, int Ho, int Wo, double *Y) {
  for (int co = 0; co < Cout; ++co)
    for (int y = 0; y < Ho; ++y)
      for (int x = 0; x < Wo; ++x) {
        double acc = bias ? (double)bias[co] : 0.0;
        for (int ci = 0; ci < Cin; ++ci)
          for (int r = 0; r < R; ++r) {
            int yi = y * stride + r - pad;
            if (yi < 0 || yi >= H) continue;
            for (int s = 0; s < S; ++s) {
              int xi = x * stride + s - pad;
              if (xi < 0 || xi >= W) continue;
              acc += (double)Wt[((size_t)(co * Cin + ci) * R + r) * S + s] *
                     X[((size_t)ci * H + yi) * W + xi];
            }
          }
        Y[((size_t)co * Ho + y) * Wo + x] = acc;
      }
}

/* Batched conv exposed for the linearity / library pins (P4, P5).
 * X [B][Cin][H][W] fp64, Y [B][Cout][Ho][Wo] fp64. */
int tac_oracle_conv2d(const double *X, const float *Wt, const float *bias,
                      int B, int Cin, int H, int W, int Cout, int R, int S,
                      int stride, int pad, double *Y) {
  int Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - S) / stride + 1;
  if (Ho < 1 || Wo < 1) return -1;
  for (int b = 0; b < B; ++b)
    conv_one(X + (size_t)b * Cin * H * W, Wt, bias, Cin, H, W, Cout, R, S,
             stride, pad, Ho, Wo, Y + (size_t)b * Cout * Ho * Wo);
  return 0;
}

/* One LIF step of one neuron.  decay = beta (dense, TAC-TP) or beta^K (TAC).
 * Returns the spike; updates *V and *s_prev.  Replay semantics documented above. */
static int lif_step(double *V, int *s_prev, double I, double decay, double v_th,
                    double v_reset, int reset, const uint8_t *dev, double band,
                    int64_t *mismatch, int64_t *excused) {
  double v = decay * (*V) + I;                       /* Alg.1 l.5 / Alg.2 l.6 */
  if (reset == OR_RESET_DELAYED) v -= v_th * (double)(*s_prev); /* Eq. (1) */
  int s = (v >= v_th) ? 1 : 0;                       /* Theta, R2 */
  if (dev) {
    int d = *dev ? 1 : 0;
    if (fabs(v - v_th) <= band) {
      s = d;
      ++*excused;
    } else if (s != d) {
      ++*mismatch;
    }
  }
  if (reset == OR_RESET_SUBTRACT) v -= (double)s * v_th; /* Alg.1 l.7 */
  else if (reset == OR_RESET_HARD) { if (s) v = v_reset; }
  *s_prev = s;
  *V = v;
  return s;
}

/*
 * Full layer forward.
 *   S        : u8 [T][B][Cin][H][W] in {0,1}
 *   Wt, bias : fp32 [Cout][Cin][R][S], [Cout] or NULL
 *   v_init   : fp64 [B][Cout][Ho][Wo] or NULL (=> 0, "Initialize V <- 0", Alg.1 l.1)
 *   out      : u8 [T_out][B][Cout][Ho][Wo], T_out = T/K (TAC) else T
 *   v_final  : fp64 [B][Cout][Ho][Wo] or NULL
 *   counts   : int64 [B][Cout] or NULL  (sum over t, y, x of out)
 *   replay   : u8, same layout as out, or NULL
 *   mismatch/excused : int64 scalars (may be NULL when replay is NULL)
 * Returns 0, or -1 on a bad argument (K not dividing T, etc.).
 */
static int forward_impl(const uint8_t *S, const double *X, const double *alpha,
                        const float *Wt, const float *bias,
                        int T, int B, int Cin, int H, int W, int Cout, int R,
                        int Sk, int stride, int pad, int K, int mode,
                        double beta, double v_th, double v_reset, int reset,
                        const double *v_init, uint8_t *out, double *v_final,
                        int64_t *counts, const uint8_t *replay, double band,
                        int64_t *mismatch_out, int64_t *excused_out) {
  if (mode == OR_MODE_DENSE) K = 1;
  const int partial = K < 0;  /* K < 0: group size -K with a partial last group (ceil) */
  if (partial) K = -K;
  if (K < 1 || T < 1 || (!partial && T % K != 0)) return -1;
  int Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - Sk) / stride + 1;
  if (Ho < 1 || Wo < 1) return -1;
  /* K | T: G = T/K groups.  Partial (reading D6'): G = ceil(T/K), the last group
   * has K_g = T - (G-1)K frames and is exactly a K = K_g group (A, decay, steps). */
  const int G = (T + K - 1) / K;
  const int T_out = (mode == OR_MODE_TAC) ? G : T;
  const size_t nin = (size_t)Cin * H * W, nout = (size_t)Cout * Ho * Wo;
  int64_t mism = 0, exc = 0;

#pragma omp parallel for schedule(dynamic, 1) reduction(+ : mism, exc)
  for (int b = 0; b < B; ++b) {
    double *A = (double *)malloc(nin * sizeof(double));
    double *Y = (double *)malloc(nout * sizeof(double));
    double *V = (double *)malloc(nout * sizeof(double));
    int *sp = (int *)malloc(nout * sizeof(int));
    for (size_t n = 0; n < nout; ++n) {
      V[n] = v_init ? v_init[(size_t)b * nout + n] : 0.0;
      sp[n] = (reset == OR_RESET_DELAYED && V[n] >= v_th) ? 1 : 0; /* R4 */
    }
    if (counts) for (int co = 0; co < Cout; ++co) counts[(size_t)b * Cout + co] = 0;

    for (int k = 0; k < G; ++k) {
      const int Kg = (T - k * K < K) ? T - k * K : K; /* frames in this group */
      /* A_k = sum_{j=0}^{K-1} beta^{K-1-j} S_{kK+j}.  Dense: A = S_t.
       * Learnable weights (reading R11): alpha_j in place of beta^{K-1-j}; a short
       * group of Kg frames takes the last Kg entries alpha[K-Kg+j] (reading D6'). */
      for (size_t i = 0; i < nin; ++i) A[i] = 0.0;
      for (int j = 0; j < Kg; ++j) {
        double wj = (alpha && mode != OR_MODE_DENSE) ? alpha[K - Kg + j]
                                                     : pow(beta, (double)(Kg - 1 - j));
        const size_t off = ((size_t)(k * K + j) * B + b) * nin;
        if (X) { /* continuous-valued input frames, same definition */
          for (size_t i = 0; i < nin; ++i) A[i] += wj * X[off + i];
        } else {
          for (size_t i = 0; i < nin; ++i) A[i] += wj * (double)S[off + i];
        }
      }
      /* Y_k = Conv2d(A_k, W): one conv call per group (Alg.1 l.4, Alg.2 l.4). */
      conv_one(A, Wt, bias, Cin, H, W, Cout, R, Sk, stride, pad, Ho, Wo, Y);

      int nsteps = (mode == OR_MODE_TACTP) ? Kg : 1;
      double decay = (mode == OR_MODE_TAC) ? pow(beta, (double)Kg) : beta;
      for (int j = 0; j < nsteps; ++j) {
        int t_out = (mode == OR_MODE_TAC) ? k : k * K + j;
        size_t ob = ((size_t)t_out * B + b) * nout;
        for (size_t n = 0; n < nout; ++n) {
          int s = lif_step(&V[n], &sp[n], Y[n], decay, v_th, v_reset, reset,
                           replay ? replay + ob + n : NULL, band, &mism, &exc);
          out[ob + n] = (uint8_t)s;
          if (counts && s) counts[(size_t)b * Cout + n / ((size_t)Ho * Wo)] += 1;
        }
      }
    }
    if (v_final) memcpy(v_final + (size_t)b * nout, V, nout * sizeof(double));
    free(A); free(Y); free(V); free(sp);
  }
  (void)T_out;
  if (mismatch_out) *mismatch_out = mism;
  if (excused_out) *excused_out = exc;
  return 0;
}

int tac_oracle_forward(const uint8_t *S, const float *Wt, const float *bias,
                       int T, int B, int Cin, int H, int W, int Cout, int R,
                       int Sk, int stride, int pad, int K, int mode,
                       double beta, double v_th, double v_reset, int reset,
                       const double *v_init, uint8_t *out, double *v_final,
                       int64_t *counts, const uint8_t *replay, double band,
                       int64_t *mismatch_out, int64_t *excused_out) {
  if (!S) return -1;
  return forward_impl(S, NULL, NULL, Wt, bias, T, B, Cin, H, W, Cout, R, Sk, stride, pad, K, mode,
                      beta, v_th, v_reset, reset, v_init, out, v_final, counts, replay, band,
                      mismatch_out, excused_out);
}

/* Same layer on continuous-valued input frames X: fp64 [T][B][Cin][H][W] (the DVS
 * network's first-layer input is log-normalised event counts; the aggregate
 * A_k = sum_j beta^{K-1-j} X_{kK+j} and everything after it are unchanged). */
int tac_oracle_forward_x(const double *X, const float *Wt, const float *bias,
                         int T, int B, int Cin, int H, int W, int Cout, int R,
                         int Sk, int stride, int pad, int K, int mode,
                         double beta, double v_th, double v_reset, int reset,
                         const double *v_init, uint8_t *out, double *v_final,
                         int64_t *counts, const uint8_t *replay, double band,
                         int64_t *mismatch_out, int64_t *excused_out) {
  if (!X) return -1;
  return forward_impl(NULL, X, NULL, Wt, bias, T, B, Cin, H, W, Cout, R, Sk, stride, pad, K, mode,
                      beta, v_th, v_reset, reset, v_init, out, v_final, counts, replay, band,
                      mismatch_out, excused_out);
}

/* Either input kind (exactly one of S, X non-NULL) with learnable aggregation weights
 * alpha [K] (fp64; NULL = beta^{K-1-j}). */
int tac_oracle_forward_alpha(const uint8_t *S, const double *X, const double *alpha,
                             const float *Wt, const float *bias,
                             int T, int B, int Cin, int H, int W, int Cout, int R,
                             int Sk, int stride, int pad, int K, int mode,
                             double beta, double v_th, double v_reset, int reset,
                             const double *v_init, uint8_t *out, double *v_final,
                             int64_t *counts, const uint8_t *replay, double band,
                             int64_t *mismatch_out, int64_t *excused_out) {
  if ((S == NULL) == (X == NULL)) return -1;
  return forward_impl(S, X, alpha, Wt, bias, T, B, Cin, H, W, Cout, R, Sk, stride, pad, K, mode,
                      beta, v_th, v_reset, reset, v_init, out, v_final, counts, replay, band,
                      mismatch_out, excused_out);
}

/* 2x2 stride-2 OR pool of binary maps (= max-pool of {0,1}, "MaxPool(2)").
 * in u8 [N][C][H][W] -> out u8 [N][C][H/2][W/2]; H, W even. */
int tac_oracle_or_pool2(const uint8_t *in, int N, int C, int H, int W, uint8_t *out) {
  if (H % 2 || W % 2) return -1;
  int Hp = H / 2, Wp = W / 2;
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c)
      for (int y = 0; y < Hp; ++y)
        for (int x = 0; x < Wp; ++x) {
          const uint8_t *p = in + (((size_t)n * C + c) * H + 2 * y) * W + 2 * x;
          out[(((size_t)n * C + c) * Hp + y) * Wp + x] =
              (uint8_t)((p[0] | p[1] | p[W] | p[W + 1]) ? 1 : 0);
        }
  return 0;
}

/* ------------------------------------------------------------------------
 * Backward pass: surrogate-gradient BPTT through the grouped LIF (SURVEY.md
 * 8(f) #3).  The paper trains every network it reports with backpropagation
 * through time and a surrogate spike derivative (App. E P:587-588:
 * fast sigmoid slope 25 for MNIST/FMNIST, arctan alpha 2 with a detached reset
 * for DVS-Gesture).  Subtract reset only (the reset the paper trains with).
 *
 * Forward (recomputed here in fp64, the order of Alg. 1 / Alg. 2 / Eq. (1)):
 *   A_k = sum_j a_j S_{kK+j} ;  Y_k = conv(A_k) + b
 *   per LIF step t of group k:  V_t = decay U_{t-1} + Y_k ;  s_t = Theta(V_t - v_th) ;
 *                               U_t = V_t - v_th s_t           (U_{-1} = v_init)
 * Surrogate: ds_t/dV_t := h(V_t - v_th) with
 *   fast sigmoid: h(u) = 1 / (alpha |u| + 1)^2          (snnTorch fast_sigmoid, slope alpha)
 *   arctan      : h(u) = (alpha/2) / (1 + (pi/2 alpha u)^2)   (snnTorch atan)
 * Detached reset: dU_t/dV_t = 1 (the reset term carries no gradient); otherwise
 * dU_t/dV_t = 1 - v_th h.
 * Backward, t = S-1 .. 0, gU = dL/dU_{S-1} = g_vfinal (0 if NULL):
 *   dV_t = (g_out_t - [!detach] v_th gU) h_t + gU ;  gY_k += dV_t ;  gU <- decay dV_t
 *   g_vinit = gU ;  g_b += sum_pixels gY_k ;  g_W += corr(gY_k, A_k) ;
 *   gA_k = conv^T(gY_k, W) ;  g_in_{kK+j} = a_j gA_k ;  g_alpha_j += <gA_k, S_{kK+j}>
 * Replay: as forward (device spikes inside the band), so the trajectory the
 * gradient is taken along is the device's.
 *   g_out   : fp64 [S][B][Cout][Ho][Wo] (dL/ds per output step; S = T_out)
 *   outputs : g_W [Cout][Cin][R][Sk], g_b [Cout] (overwritten); g_in [T][B][Cin][H][W],
 *             g_vinit [B][Cout][Ho][Wo], g_alpha [K]: each may be NULL.
 * K must divide T (no partial groups).  Returns 0 or -1.
 * ------------------------------------------------------------------------ */
static double surrogate(int kind, double a, double u) {
  if (kind == 0) {
    const double d = a * fabs(u) + 1.0;
    return 1.0 / (d * d);
  }
  const double z = 1.5707963267948966 * a * u;
  return 0.5 * a / (1.0 + z * z);
}

int tac_oracle_backward(const uint8_t *S, const double *X, const double *alpha,
                        const float *Wt, const float *bias,
                        int T, int B, int Cin, int H, int W, int Cout, int R, int Sk,
                        int stride, int pad, int K, int mode, double beta, double v_th,
                        int sg_kind, double sg_alpha, int detach,
                        const double *v_init, const uint8_t *replay, double band,
                        const double *g_out, const double *g_vfinal,
                        double *g_W, double *g_b, double *g_in, double *g_vinit, double *g_alpha) {
  if ((S == NULL) == (X == NULL) || !g_out || !g_W || !g_b) return -1;
  if (mode == OR_MODE_DENSE) K = 1;
  if (K < 1 || T < 1 || T % K != 0) return -1;
  const int Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - Sk) / stride + 1;
  if (Ho < 1 || Wo < 1) return -1;
  const int G = T / K;
  const int ns = (mode == OR_MODE_TACTP) ? K : 1;
  const int Sout = G * ns;
  const double decay = (mode == OR_MODE_TAC) ? pow(beta, (double)K) : beta;
  const size_t nin = (size_t)Cin * H * W, nout = (size_t)Cout * Ho * Wo, nw = (size_t)Cout * Cin * R * Sk;
  double *aj = (double *)malloc((size_t)K * sizeof(double));
  for (int j = 0; j < K; ++j)
    aj[j] = (alpha && mode != OR_MODE_DENSE) ? alpha[j] : pow(beta, (double)(K - 1 - j));
  for (size_t i = 0; i < nw; ++i) g_W[i] = 0.0;
  for (int co = 0; co < Cout; ++co) g_b[co] = 0.0;
  if (g_alpha) for (int j = 0; j < K; ++j) g_alpha[j] = 0.0;
  int rc = 0;
  for (int b = 0; b < B; ++b) {   /* sequential over samples: the gradients are sums over b */
    double *A = (double *)malloc((size_t)G * nin * sizeof(double));
    double *Vp = (double *)malloc((size_t)Sout * nout * sizeof(double));
    double *Y = (double *)malloc(nout * sizeof(double));
    double *gY = (double *)malloc((size_t)G * nout * sizeof(double));
    double *gU = (double *)malloc(nout * sizeof(double));
    double *U = (double *)malloc(nout * sizeof(double));
    double *gA = (double *)malloc(nin * sizeof(double));
    if (!A || !Vp || !Y || !gY || !gU || !U || !gA) { rc = -1; goto done_b; }
    /* forward recompute */
    for (size_t n = 0; n < nout; ++n) U[n] = v_init ? v_init[(size_t)b * nout + n] : 0.0;
    for (int k = 0; k < G; ++k) {
      double *Ak = A + (size_t)k * nin;
      for (size_t i = 0; i < nin; ++i) Ak[i] = 0.0;
      for (int j = 0; j < K; ++j) {
        const size_t off = ((size_t)(k * K + j) * B + b) * nin;
        for (size_t i = 0; i < nin; ++i) Ak[i] += aj[j] * (X ? X[off + i] : (double)S[off + i]);
      }
      conv_one(Ak, Wt, bias, Cin, H, W, Cout, R, Sk, stride, pad, Ho, Wo, Y);
      for (int j = 0; j < ns; ++j) {
        const int t = k * ns + j;
        const size_t ob = ((size_t)t * B + b) * nout;
        for (size_t n = 0; n < nout; ++n) {
          const double v = decay * U[n] + Y[n];
          int s = v >= v_th;
          if (replay && fabs(v - v_th) <= band) s = replay[ob + n] ? 1 : 0;
          Vp[(size_t)t * nout + n] = v;
          U[n] = v - v_th * (double)s;
        }
      }
    }
    /* BPTT through the LIF steps, latest first */
    for (size_t n = 0; n < nout; ++n) gU[n] = g_vfinal ? g_vfinal[(size_t)b * nout + n] : 0.0;
    for (size_t i = 0; i < (size_t)G * nout; ++i) gY[i] = 0.0;
    for (int t = Sout - 1; t >= 0; --t) {
      const int k = t / ns;
      const size_t ob = ((size_t)t * B + b) * nout;
      for (size_t n = 0; n < nout; ++n) {
        const double h = surrogate(sg_kind, sg_alpha, Vp[(size_t)t * nout + n] - v_th);
        const double dV = (g_out[ob + n] - (detach ? 0.0 : v_th * gU[n])) * h + gU[n];
        gY[(size_t)k * nout + n] += dV;
        gU[n] = decay * dV;
      }
    }
    if (g_vinit) memcpy(g_vinit + (size_t)b * nout, gU, nout * sizeof(double));
    /* the group convolution's gradients */
    for (int k = 0; k < G; ++k) {
      const double *gYk = gY + (size_t)k * nout, *Ak = A + (size_t)k * nin;
      for (int co = 0; co < Cout; ++co)
        for (int y = 0; y < Ho; ++y)
          for (int x = 0; x < Wo; ++x) {
            const double g = gYk[((size_t)co * Ho + y) * Wo + x];
            g_b[co] += g;
            for (int ci = 0; ci < Cin; ++ci)
              for (int r = 0; r < R; ++r) {
                const int yi = y * stride + r - pad;
                if (yi < 0 || yi >= H) continue;
                for (int s = 0; s < Sk; ++s) {
                  const int xi = x * stride + s - pad;
                  if (xi < 0 || xi >= W) continue;
                  g_W[((size_t)(co * Cin + ci) * R + r) * Sk + s] += g * Ak[((size_t)ci * H + yi) * W + xi];
                }
              }
          }
      if (!g_in && !g_alpha) continue;
      for (size_t i = 0; i < nin; ++i) gA[i] = 0.0;
      for (int co = 0; co < Cout; ++co)
        for (int y = 0; y < Ho; ++y)
          for (int x = 0; x < Wo; ++x) {
            const double g = gYk[((size_t)co * Ho + y) * Wo + x];
            for (int ci = 0; ci < Cin; ++ci)
              for (int r = 0; r < R; ++r) {
                const int yi = y * stride + r - pad;
                if (yi < 0 || yi >= H) continue;
                for (int s = 0; s < Sk; ++s) {
                  const int xi = x * stride + s - pad;
                  if (xi < 0 || xi >= W) continue;
                  gA[((size_t)ci * H + yi) * W + xi] += g * (double)Wt[((size_t)(co * Cin + ci) * R + r) * Sk + s];
                }
              }
          }
      for (int j = 0; j < K; ++j) {
        const size_t off = ((size_t)(k * K + j) * B + b) * nin;
        if (g_in)
          for (size_t i = 0; i < nin; ++i) g_in[off + i] = aj[j] * gA[i];
        if (g_alpha && alpha && mode != OR_MODE_DENSE) {
          double acc = 0.0;
          for (size_t i = 0; i < nin; ++i) acc += gA[i] * (X ? X[off + i] : (double)S[off + i]);
          g_alpha[j] += acc;
        }
      }
    }
  done_b:
    free(A); free(Vp); free(Y); free(gY); free(gU); free(U); free(gA);
    if (rc) break;
  }
  free(aj);
  return rc;
}
