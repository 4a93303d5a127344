// ViT training executor: the B200 realisation of the reference's modeled
// F / B / U blocks (schedule.cpp:40-52, 184-193) for a stage that runs the
// whole stack (K = 1) or a span of ATT/MLP sublayers (pipeline stages).
//
// Host C++ that launches the sm_100a kernels in this library; all memory is
// caller-owned (a parameter arena and an activation workspace sized by
// eps_vit_layout / eps_vit_workspace_bytes).  Freeze semantics follow the
// reference's partition of the stack (model.cpp:79-92):
//   * layers [0, L_frozen) are frozen: forward only, no stash needed, no
//     backward, no optimizer update;
//   * with AutoCache the frozen prefix is not run at all: the boundary
//     activation X[L_frozen] is gathered from the HBM store by sample id;
//     on a boundary move the delta [old, new) is forwarded once and the new
//     boundary scattered back (autocache.cpp:45-67);
//   * the lowest trainable layer skips its input-gradient write.
// Parameter arena order = the reference's ModelSpec order, so each layer's
// tensors are one contiguous segment (embed folded into layer 0, final LN +
// head into layer L-1, model.cpp:137-142) -- the freeze test reduces those
// segments and the optimizer walks one contiguous tail [layer L_f, end).
#include <cuda_runtime.h>

#include <cstdlib>

#include <cmath>
#include <cstring>
#include <new>
#include <stdexcept>
#include <vector>

#include "eps_capi.h"

namespace {

struct Slot {
  int64_t off = 0;
  int64_t n = 0;
};

struct LayerSlots {
  Slot ln1g, ln1b, wqkv, bqkv, wp, bp;  // ATT sublayer
  Slot ln2g, ln2b, w1, b1, w2, b2;      // MLP sublayer
};

struct Geometry {
  int layers, d, f, heads, tokens, classes, image, in_image, patch, channels, max_batch;
  int classes_pad;  // head rows padded to a multiple of 8 (16 B TMA row pitch)
  int patches() const { return (image / patch) * (image / patch); }
  int patch_len() const { return channels * patch * patch; }
  int head_dim() const { return d / heads; }
};

constexpr int64_t kAlign = 64;  // elements: 256 B for fp32, 128 B for bf16

struct Layout {
  Slot wpe, bpe, cls, pos;
  std::vector<LayerSlots> layer;
  Slot lnfg, lnfb, wh, bh;
  std::vector<int64_t> seg;  // L+1 segment boundaries (freeze test / optimizer)
  int64_t total = 0;

  explicit Layout(const Geometry& g) {
    int64_t at = 0;
    auto take = [&](int64_t n) {
      Slot s{at, n};
      at += (n + kAlign - 1) / kAlign * kAlign;
      return s;
    };
    const int64_t d = g.d, f = g.f;
    seg.push_back(0);
    wpe = take(d * g.patch_len());
    bpe = take(d);
    cls = take(d);
    pos = take(int64_t(g.tokens) * d);
    layer.resize(g.layers);
    for (int l = 0; l < g.layers; ++l) {
      if (l > 0) seg.push_back(at);
      LayerSlots& s = layer[l];
      s.ln1g = take(d);
      s.ln1b = take(d);
      s.wqkv = take(3 * d * d);
      s.bqkv = take(3 * d);
      s.wp = take(d * d);
      s.bp = take(d);
      s.ln2g = take(d);
      s.ln2b = take(d);
      s.w1 = take(f * d);
      s.b1 = take(f);
      s.w2 = take(d * f);
      s.b2 = take(d);
    }
    lnfg = take(d);
    lnfb = take(d);
    wh = take(int64_t(g.classes_pad) * d);
    bh = take(g.classes_pad);
    total = at;
    seg.push_back(total);
  }
};

// Activation workspace carve (all [rows, width] bf16 unless noted).
struct Acts {
  std::vector<uint16_t*> X, H1, QKV, A, X1, H2, U, G;
  std::vector<float*> mean1, rstd1, mean2, rstd2, lse;
  uint16_t *patches = nullptr, *ptok = nullptr, *cls_rows = nullptr, *hf = nullptr,
           *logits = nullptr, *dlogits = nullptr, *dhf = nullptr, *dcls = nullptr;
  float *meanf = nullptr, *rstdf = nullptr;
  uint16_t *dX = nullptr, *dH = nullptr, *dA = nullptr, *dQKV = nullptr, *dptok = nullptr;
  float* dsum = nullptr;
  float* drow = nullptr;  // attention D = rowsum(dO * O) [rows, heads] (ROWDOT epilogue)
  double* sq_ws = nullptr;
  size_t sq_ws_bytes = 0;
  size_t bytes = 0;

  Acts(const Geometry& g, int64_t param_total, uint8_t* base) {
    const int64_t R = int64_t(g.max_batch) * g.tokens, d = g.d, f = g.f, L = g.layers;
    const int64_t B = g.max_batch, BP = B * g.patches();
    size_t at = 0;
    auto take = [&](size_t bytes) {
      uint8_t* p = base ? base + at : nullptr;
      at += (bytes + 255) / 256 * 256;
      return p;
    };
    auto bf = [&](int64_t n) { return reinterpret_cast<uint16_t*>(take(size_t(n) * 2)); };
    auto fp = [&](int64_t n) { return reinterpret_cast<float*>(take(size_t(n) * 4)); };
    for (int64_t l = 0; l <= L; ++l) X.push_back(bf(R * d));
    for (int64_t l = 0; l < L; ++l) {
      H1.push_back(bf(R * d));
      QKV.push_back(bf(R * 3 * d));
      A.push_back(bf(R * d));
      X1.push_back(bf(R * d));
      H2.push_back(bf(R * d));
      U.push_back(bf(R * f));
      G.push_back(bf(R * f));
      mean1.push_back(fp(R));
      rstd1.push_back(fp(R));
      mean2.push_back(fp(R));
      rstd2.push_back(fp(R));
      lse.push_back(fp(B * g.heads * g.tokens));
    }
    patches = bf(BP * g.patch_len());
    ptok = bf(BP * d);
    cls_rows = bf(B * d);
    hf = bf(B * d);
    logits = bf(B * g.classes_pad);
    dlogits = bf(B * g.classes_pad);
    dhf = bf(B * d);
    dcls = bf(B * d);
    meanf = fp(B);
    rstdf = fp(B);
    dX = bf(R * d);
    dH = bf(R * d);
    dA = bf(R * d);
    dQKV = bf(R * 3 * d);
    dptok = bf(BP * d);
    dsum = fp(B * g.heads * g.tokens);
    drow = fp(B * g.heads * g.tokens);
    sq_ws_bytes = size_t((param_total + 65535) / 65536 + 64) * 8;
    sq_ws = reinterpret_cast<double*>(take(sq_ws_bytes));
    bytes = at;
  }
};

int check(int rc) {
  if (rc != EPS_OK) throw rc;
  return rc;
}

}  // namespace

struct eps_vit {
  Geometry g;
  Layout lay;
  Acts act;
  float* p32;
  uint16_t* p16;
  float* g32;
  float* mom;
  float* loss_sum;  // device scalar owned by caller
  // Stage hand-off over peer memory: the output cut `out_g` is written to
  // `out_to` (the next stage's buffer) and the gradient at the input cut
  // `dx_g` to `dx_to` (the previous stage's dX), both [max_batch*T, d].
  int out_g = -1, dx_g = -1;
  // AutoCache store sharded over the node's GPUs (eps_cache_gather_sharded):
  // device table of shard base pointers; null = one local / host store.
  const uint64_t* shard_table = nullptr;
  int64_t rows_per_shard = 0;
  uint16_t* out_to = nullptr;
  uint16_t* dx_to = nullptr;
  uint16_t* out_buf(int gs, uint16_t* local) const {
    return (gs == out_g && out_to != nullptr) ? out_to : local;
  }
  uint16_t* dx_buf(int gs) const { return (gs == dx_g && dx_to != nullptr) ? dx_to : act.dX; }
  eps_vit(const Geometry& geom, float* p, uint16_t* pb, float* gr, float* m, uint8_t* ws)
      : g(geom), lay(geom), act(geom, lay.total, ws), p32(p), p16(pb), g32(gr), mom(m),
        loss_sum(nullptr) {
    if (side_stream_on()) {
      cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming);
    }
  }
  ~eps_vit() {
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    if (side) {
      cudaStreamSynchronize(side);
      cudaStreamDestroy(side);
      cudaEventDestroy(fork_ev);
      cudaEventDestroy(join_ev);
    }
  }

  // ---- weight gradients on a side stream ----------------------------------------
  // A weight-gradient GEMM only reads its inputs and accumulates into g32, so
  // it can run beside the input-gradient chain: fork() makes the side stream
  // wait for the main stream's work so far, join() makes the main stream wait
  // for the side stream.  Small micro-batches (K = 8 pipeline stages) leave
  // most SMs idle during each GEMM; the side stream fills them.
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  static bool side_stream_on() {
    static const bool on = [] {
      const char* e = std::getenv("EPS_SIDE_STREAM");
      return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
  }
  bool side_on = true;  // eps_vit_set_side_stream
  // (off while per-class timing is on: concurrent kernels would make the
  // class durations overlap and overstate the GEMM class time)
  cudaStream_t fork(cudaStream_t st) {
    if (!side || !side_on || timing) return st;
    cudaEventRecord(fork_ev, st);
    cudaStreamWaitEvent(side, fork_ev, 0);
    return side;
  }
  void join(cudaStream_t st) {
    if (!side || !side_on || timing) return;
    cudaEventRecord(join_ev, side);
    cudaStreamWaitEvent(st, join_ev, 0);
  }

  // ---- per-class launch timing (eps_vit_timing_*) ----------------------------
  struct Rec {
    int cls;
    double flops, bytes;
    cudaEvent_t a, b;
  };
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<Rec> recs;
  cudaEvent_t next_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) throw int(EPS_ECUDA);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  // Run one C-ABI launch; when timing, bracket it with events on `st`.
  template <typename F>
  void run(int cls, double flops, double bytes, cudaStream_t st, F&& launch) {
    if (!timing) {
      check(launch());
      return;
    }
    Rec r{cls, flops, bytes, next_event(), next_event()};
    cudaEventRecord(r.a, st);
    check(launch());
    cudaEventRecord(r.b, st);
    recs.push_back(r);
  }
  // GEMM with algorithmic FLOPs 2MNK.
  void mm(int a_mn, int b_mn, int epi, const void* A, const void* B, void* C, const float* bias,
          void* aux, float* colsum, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
          int64_t ldc, int split, cudaStream_t st) {
    run(EPS_TC_GEMM, 2.0 * double(M) * double(N) * double(K), 0.0, st, [&] {
      return eps_gemm_bf16(a_mn, b_mn, epi, A, B, C, bias, aux, colsum, M, N, K, lda, ldb, ldc,
                           split, st);
    });
  }
  void layernorm(const uint16_t* x, const Slot& gam, const Slot& bet, uint16_t* y, float* mean,
                 float* rstd, int64_t rows, cudaStream_t st) {
    run(EPS_TC_NORM, 0.0, 4.0 * double(rows) * g.d, st, [&] {
      return eps_layernorm_fwd(x, P(gam), P(bet), y, mean, rstd, rows, g.d, 1e-6f, st);
    });
  }
  void layernorm_bwd(const uint16_t* dy, const uint16_t* x, const Slot& gam, const Slot& bet,
                     const float* mean, const float* rstd, const uint16_t* dres, uint16_t* dx,
                     float* colsum_dx, int64_t rows, cudaStream_t st) {
    run(EPS_TC_NORM, 0.0, 8.0 * double(rows) * g.d, st, [&] {
      return eps_layernorm_bwd(dy, x, P(gam), mean, rstd, dres, dx, Gr(gam), Gr(bet), colsum_dx,
                               rows, g.d, nullptr, st);
    });
  }
  template <typename F>
  void eltwise(cudaStream_t st, F&& launch) {
    run(EPS_TC_ELTWISE, 0.0, 0.0, st, launch);
  }

  const uint16_t* W(const Slot& s) const { return p16 + s.off; }
  const float* P(const Slot& s) const { return p32 + s.off; }
  float* Gr(const Slot& s) const { return g32 + s.off; }
  float scale() const { return 1.0f / std::sqrt(float(g.head_dim())); }
  int64_t row_bytes() const { return int64_t(g.tokens) * g.d * 2; }

  int split_for(int64_t rows) const {
    // wgrad contracts over the token rows; split so the grid covers the SMs
    return rows >= 16384 ? 8 : rows >= 4096 ? 4 : 1;
  }

  // ---- sublayer geometry ------------------------------------------------------
  // Global sublayer g in [0, 2L): layer g/2, ATT if even, MLP if odd
  // (the reference's SublayerSeq order, model.hpp:56-74).
  // Residual-stream buffer at the cut *before* sublayer g.
  uint16_t* cut(int gs) const {
    if (gs >= 2 * g.layers) return act.X[g.layers];
    return (gs % 2 == 0) ? act.X[gs / 2] : act.X1[gs / 2];
  }
  // Bias whose gradient is the column sum of dL/d(output of sublayer g).
  float* out_bias_grad(int gs) const {
    const LayerSlots& s = lay.layer[gs / 2];
    return (gs % 2 == 0) ? Gr(s.bp) : Gr(s.b2);
  }
  // Parameter elements of sublayer g: ATT = [seg[l], ln2g), MLP = [ln2g, seg[l+1]);
  // the embedding folds into sublayer 0, the final LN + head into 2L-1.
  int64_t sub_begin(int gs) const {
    if (gs >= 2 * g.layers) return lay.total;
    return (gs % 2 == 0) ? lay.seg[gs / 2] : lay.layer[gs / 2].ln2g.off;
  }

  // ---- forward sublayers on rows [r0, r0+R) / samples [b0, b0+b) -----------
  void embed_fwd(const float* images, int b0, int b, cudaStream_t st) {
    const int64_t d = g.d, np = g.patches(), pl = g.patch_len();
    uint16_t* patches = act.patches + int64_t(b0) * np * pl;
    uint16_t* ptok = act.ptok + int64_t(b0) * np * d;
    const int img_arg = (g.in_image != g.image) ? ((g.in_image << 16) | g.image) : g.image;
    const float* img = images + int64_t(b0) * g.channels * g.in_image * g.in_image;
    eltwise(st, [&] { return eps_patchify(img, patches, b, g.channels, img_arg, g.patch, st); });
    mm(0, 0, EPS_EPI_BIAS_BF16, patches, W(lay.wpe), ptok, P(lay.bpe), nullptr, nullptr, b * np,
       d, pl, pl, pl, d, 1, st);
    uint16_t* x0 = act.X[0] + int64_t(b0) * g.tokens * d;
    eltwise(st, [&] {
      return eps_vit_assemble(ptok, P(lay.cls), P(lay.pos), x0, b, g.tokens, d, st);
    });
  }

  void att_fwd(int l, int b0, int b, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    layernorm(act.X[l] + r0 * d, s.ln1g, s.ln1b, act.H1[l] + r0 * d, act.mean1[l] + r0,
              act.rstd1[l] + r0, R, st);
    mm(0, 0, EPS_EPI_BIAS_BF16, act.H1[l] + r0 * d, W(s.wqkv), act.QKV[l] + r0 * 3 * d,
       P(s.bqkv), nullptr, nullptr, R, 3 * d, d, d, d, 3 * d, 1, st);
    const double t = g.tokens, hd = double(g.heads) * g.head_dim();
    run(EPS_TC_ATTN, 4.0 * b * t * t * hd, 8.0 * b * t * hd, st, [&] {
      return eps_attn_fwd(act.QKV[l] + r0 * 3 * d, act.A[l] + r0 * d,
                          act.lse[l] + int64_t(b0) * g.heads * g.tokens, b, g.tokens, g.heads,
                          g.head_dim(), scale(), st);
    });
    mm(0, 0, EPS_EPI_BIAS_RESID_BF16, act.A[l] + r0 * d, W(s.wp),
       out_buf(2 * l + 1, act.X1[l]) + r0 * d, P(s.bp), act.X[l] + r0 * d, nullptr, R, d, d, d,
       d, d, 1, st);
  }

  void mlp_fwd(int l, int b0, int b, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, f = g.f, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    layernorm(act.X1[l] + r0 * d, s.ln2g, s.ln2b, act.H2[l] + r0 * d, act.mean2[l] + r0,
              act.rstd2[l] + r0, R, st);
    mm(0, 0, EPS_EPI_BIAS_GELU2_BF16, act.H2[l] + r0 * d, W(s.w1), act.G[l] + r0 * f, P(s.b1),
       act.U[l] + r0 * f, nullptr, R, f, d, d, d, f, 1, st);
    mm(0, 0, EPS_EPI_BIAS_RESID_BF16, act.G[l] + r0 * f, W(s.w2),
       out_buf(2 * l + 2, act.X[l + 1]) + r0 * d, P(s.b2), act.X1[l] + r0 * d, nullptr, R, d, f,
       f, f, d, 1, st);
  }

  void sub_fwd(int gs, int b0, int b, cudaStream_t st) {
    if (gs % 2 == 0) att_fwd(gs / 2, b0, b, st);
    else mlp_fwd(gs / 2, b0, b, st);
  }

  // Head forward + loss + head backward; leaves dL/dX[L] in act.dX rows.
  void head_fwd_bwd(const int64_t* labels, int b0, int b, int global_batch, cudaStream_t st) {
    const int64_t d = g.d, C = g.classes_pad, T = g.tokens;
    const LayerSlots& top = lay.layer[g.layers - 1];
    uint16_t* cls = act.cls_rows + int64_t(b0) * d;
    uint16_t* hf = act.hf + int64_t(b0) * d;
    uint16_t* logits = act.logits + int64_t(b0) * C;
    uint16_t* dlogits = act.dlogits + int64_t(b0) * C;
    uint16_t* dhf = act.dhf + int64_t(b0) * d;
    uint16_t* dcls = act.dcls + int64_t(b0) * d;
    const uint16_t* xl = act.X[g.layers] + int64_t(b0) * T * d;
    eltwise(st, [&] { return eps_gather_rows(xl, T * d, cls, b, d, 0, st); });
    layernorm(cls, lay.lnfg, lay.lnfb, hf, act.meanf + b0, act.rstdf + b0, b, st);
    mm(0, 0, EPS_EPI_BIAS_BF16, hf, W(lay.wh), logits, P(lay.bh), nullptr, nullptr, b, C, d, d, d,
       C, 1, st);
    eltwise(st, [&] {
      return eps_softmax_xent_bias(logits, labels + b0, dlogits, loss_sum, Gr(lay.bh), b,
                                   g.classes, int(C), 1.0f / float(global_batch), st);
    });
    mm(1, 1, EPS_EPI_ACCUM_F32, dlogits, hf, Gr(lay.wh), nullptr, nullptr, nullptr, C, d, b, C, d,
       d, 1, st);
    mm(0, 1, EPS_EPI_STORE_BF16, dlogits, W(lay.wh), dhf, nullptr, nullptr, nullptr, b, d, C, C,
       d, d, 1, st);
    // LN_f backward on the CLS rows; its dx column sum is top-layer FC2's bias grad
    layernorm_bwd(dhf, cls, lay.lnfg, lay.lnfb, act.meanf + b0, act.rstdf + b0, nullptr, dcls,
                  Gr(top.b2), b, st);
    uint16_t* dX = act.dX + int64_t(b0) * T * d;
    if (cudaMemsetAsync(dX, 0, size_t(b) * T * d * 2, st) != cudaSuccess) throw int(EPS_ECUDA);
    eltwise(st, [&] { return eps_scatter_rows(dcls, dX, T * d, b, d, 0, st); });
  }

  // ---- backward sublayers (dX holds dL/d(output) rows; updated in place) ----
  // colsum_prev: bias grad of the sublayer that produced this sublayer's input
  // (accumulated from the fused LN backward), or null when that producer
  // lives on another pipeline stage (the receiver computes it there).
  void mlp_bwd(int l, int b0, int b, float* colsum_prev, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, f = g.f, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    uint16_t* dX = act.dX + r0 * d;
    uint16_t* Gm = act.G[l] + r0 * f;
    const int split = 0;  // auto split-K (eps_gemm_bf16)
    mm(1, 1, EPS_EPI_ACCUM_F32, dX, Gm, Gr(s.w2), nullptr, nullptr, nullptr, d, f, R, d, f, f,
       split, st);
    // du overwrites G (its last reader was the dW2 GEMM above)
    mm(0, 1, EPS_EPI_MUL_BF16, dX, W(s.w2), Gm, nullptr, act.U[l] + r0 * f, Gr(s.b1), R, f, d,
       d, f, f, 1, st);
    // dW1 (reads du, H2) beside dH = du W1 and the LayerNorm backward
    mm(1, 1, EPS_EPI_ACCUM_F32, Gm, act.H2[l] + r0 * d, Gr(s.w1), nullptr, nullptr, nullptr, f,
       d, R, f, d, d, split, fork(st));
    mm(0, 1, EPS_EPI_STORE_BF16, Gm, W(s.w1), act.dH + r0 * d, nullptr, nullptr, nullptr, R, d,
       f, f, d, d, 1, st);
    layernorm_bwd(act.dH + r0 * d, act.X1[l] + r0 * d, s.ln2g, s.ln2b, act.mean2[l] + r0,
                  act.rstd2[l] + r0, dX, dx_buf(2 * l + 1) + r0 * d, colsum_prev, R, st);
    join(st);  // du (G) is overwritten by the next layer's backward
  }

  // need_dx: write dL/dX[l] (false for the lowest trainable layer when the
  // layers below are frozen).
  void att_bwd(int l, int b0, int b, bool need_dx, float* colsum_prev, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    uint16_t* dX = act.dX + r0 * d;
    const int split = 0;  // auto split-K (eps_gemm_bf16)
    // dW_o (reads dX, A) beside dA and the attention backward
    mm(1, 1, EPS_EPI_ACCUM_F32, dX, act.A[l] + r0 * d, Gr(s.wp), nullptr, nullptr, nullptr, d, d,
       R, d, d, d, split, fork(st));
    // dA = dX1 W_o; for the fused attention backward its epilogue also forms
    // D = rowsum(dA * A) per (row, head) (EPS_EPI_ROWDOT_BF16)
    const bool rowdot = eps_attn_bwd_uses_rowdot(g.tokens, g.head_dim()) != 0;
    float* drow = act.drow + r0 * g.heads;
    if (rowdot) cudaMemsetAsync(drow, 0, size_t(R) * g.heads * sizeof(float), st);
    mm(0, 1, rowdot ? EPS_EPI_ROWDOT_BF16 : EPS_EPI_STORE_BF16, dX, W(s.wp), act.dA + r0 * d,
       nullptr, rowdot ? act.A[l] + r0 * d : nullptr, rowdot ? drow : nullptr, R, d, d, d, d, d, 1,
       st);
    const double t = g.tokens, hd = double(g.heads) * g.head_dim();
    run(EPS_TC_ATTN, 8.0 * b * t * t * hd, 18.0 * b * t * hd, st, [&] {
      return eps_attn_bwd_rowdot(act.QKV[l] + r0 * 3 * d, act.A[l] + r0 * d, act.dA + r0 * d,
                                 act.lse[l] + int64_t(b0) * g.heads * g.tokens, drow,
                                 act.dQKV + r0 * 3 * d, Gr(s.bqkv),
                                 act.dsum + int64_t(b0) * g.heads * g.tokens, b, g.tokens,
                                 g.heads, g.head_dim(), scale(), st);
    });
    // dW_qkv (reads dQKV, H1) beside dH = dQKV W_qkv
    mm(1, 1, EPS_EPI_ACCUM_F32, act.dQKV + r0 * 3 * d, act.H1[l] + r0 * d, Gr(s.wqkv), nullptr,
       nullptr, nullptr, 3 * d, d, R, 3 * d, d, d, split, fork(st));
    mm(0, 1, EPS_EPI_STORE_BF16, act.dQKV + r0 * 3 * d, W(s.wqkv), act.dH + r0 * d, nullptr,
       nullptr, nullptr, R, d, 3 * d, 3 * d, d, d, 1, st);
    join(st);  // dW_o read dX, which the LayerNorm backward rewrites in place
    layernorm_bwd(act.dH + r0 * d, act.X[l] + r0 * d, s.ln1g, s.ln1b, act.mean1[l] + r0,
                  act.rstd1[l] + r0, dX, need_dx ? dx_buf(2 * l) + r0 * d : nullptr,
                  need_dx ? colsum_prev : nullptr, R, st);
  }

  void embed_bwd(int b0, int b, cudaStream_t st) {
    const int64_t d = g.d, np = g.patches(), pl = g.patch_len();
    uint16_t* dptok = act.dptok + int64_t(b0) * np * d;
    const uint16_t* dx0 = act.dX + int64_t(b0) * g.tokens * d;
    eltwise(st, [&] {
      return eps_vit_assemble_bwd(dx0, Gr(lay.cls), Gr(lay.pos), dptok, b, g.tokens, d, st);
    });
    eltwise(st, [&] { return eps_colsum_bf16(dptok, Gr(lay.bpe), int64_t(b) * np, d, st); });
    mm(1, 1, EPS_EPI_ACCUM_F32, dptok, act.patches + int64_t(b0) * np * pl, Gr(lay.wpe), nullptr,
       nullptr, nullptr, d, pl, int64_t(b) * np, d, pl, pl, 0, st);
  }

  // Backward of sublayer gs; `first` = lowest sublayer held by this stage.
  void sub_bwd(int gs, int b0, int b, int l_frozen, bool first, cudaStream_t st) {
    const int l = gs / 2;
    if (gs % 2 == 1) {
      mlp_bwd(l, b0, b, first ? nullptr : Gr(lay.layer[l].bp), st);
    } else {
      const bool need_dx = l > l_frozen || l == 0;
      float* prev = (l > 0 && !first) ? Gr(lay.layer[l - 1].b2) : nullptr;
      att_bwd(l, b0, b, need_dx, prev, st);
    }
  }

  // ---- pipeline-stage operations ------------------------------------------------
  // Forward of global sublayers [g0, g1) for samples [b0, b0+b).  `front`: this
  // stage produces its own input (pipeline stage 0): frozen prefix, AutoCache
  // gather / boundary move and the embedding run first.
  //   cache_mode 0: frozen prefix [0, L_f) recomputed forward-only;
  //   cache_mode 1: X[L_f] gathered from the store rows `ids` (prefix skipped);
  //   cache_mode 2: boundary move old -> L_f: X[old] gathered (old > 0) or
  //                 computed from the images, [old, L_f) forwarded once, X[L_f]
  //                 scattered into the store (autocache.cpp:45-67);
  //   cache_mode 3: the boundary trails L_f (the cache stays on at its old
  //                 boundary when the policy no longer wants a move,
  //                 runner.cpp:186-213): X[old] gathered, [old, L_f)
  //                 forwarded, nothing written.
  void stage_fwd(const float* images, int b0, int b, int g0, int g1, int l_frozen, bool front,
                 int cache_mode, int cache_old, void* store, const int64_t* ids,
                 cudaStream_t st) {
    const int64_t xoff = int64_t(b0) * g.tokens * g.d;
    const int64_t rb = row_bytes();
    auto cache_io = [&](bool gather, uint16_t* x) {
      run(EPS_TC_CACHE, 0.0, 2.0 * b * double(rb), st, [&] {
        if (shard_table != nullptr)
          return gather ? eps_cache_gather_sharded(shard_table, rows_per_shard, ids + b0, b, rb,
                                                   x + xoff, st)
                        : eps_cache_scatter_sharded(shard_table, rows_per_shard, ids + b0, b, rb,
                                                    x + xoff, st);
        return gather ? eps_cache_gather(store, ids + b0, b, rb, x + xoff, st)
                      : eps_cache_scatter(store, ids + b0, b, rb, x + xoff, st);
      });
    };
    if (front) {
      int start = 0;  // first frozen layer to run forward
      if (cache_mode == 1) {
        cache_io(true, act.X[l_frozen]);
        start = l_frozen;
      } else if ((cache_mode == 2 || cache_mode == 3) && cache_old > 0) {
        cache_io(true, act.X[cache_old]);
        start = cache_old;
      }
      if (start == 0 && cache_mode != 1) embed_fwd(images, b0, b, st);
      // frozen layers below the span (a span starting below 2*L_f -- AutoPipe
      // off, frozen layers on their stage -- runs them itself)
      const int prefix_end = g0 / 2 < l_frozen ? g0 / 2 : l_frozen;
      for (int l = start; l < prefix_end; ++l) {
        att_fwd(l, b0, b, st);
        mlp_fwd(l, b0, b, st);
      }
      if (cache_mode == 2) cache_io(false, act.X[l_frozen]);
    }
    for (int gs = g0; gs < g1; ++gs) sub_fwd(gs, b0, b, st);
  }

  // Backward of [g0, g1) in reverse with dL/d(output of g1-1) in dX rows.
  // cut_out: that gradient arrived from the next stage, so this stage also
  // owns the column sum for sublayer g1-1's output bias.
  // Sublayers [g0, g1) of a stage whose lowest sublayer is stage_g0 (the host
  // may walk a stage's span in pieces, e.g. to launch gradient buckets early).
  void stage_bwd(int b0, int b, int g0, int g1, int stage_g0, int l_frozen, bool cut_out,
                 cudaStream_t st) {
    // frozen sublayers inside the span have no backward
    if (g0 < 2 * l_frozen) g0 = 2 * l_frozen;
    if (stage_g0 < 2 * l_frozen) stage_g0 = 2 * l_frozen;
    if (g1 <= g0) return;
    const int64_t d = g.d, R = int64_t(b) * g.tokens;
    if (cut_out) {
      const uint16_t* dx = act.dX + int64_t(b0) * g.tokens * d;
      float* bias = out_bias_grad(g1 - 1);
      eltwise(st, [&] { return eps_colsum_bf16(dx, bias, R, d, st); });
    }
    for (int gs = g1 - 1; gs >= g0; --gs) sub_bwd(gs, b0, b, l_frozen, gs == stage_g0, st);
    if (g0 == 0 && l_frozen == 0) embed_bwd(b0, b, st);
  }

  void sgd_range(int64_t begin, int64_t end, float lr, float mu, float wd, cudaStream_t st) {
    if (end <= begin) return;
    run(EPS_TC_OPTIM, 0.0, 26.0 * double(end - begin), st, [&] {
      return eps_sgd_momentum(p32 + begin, p16 + begin, g32 + begin, mom + begin, end - begin, lr,
                              mu, wd, st);
    });
  }

  void sqnorm_ranges(const int64_t* offsets, int n, double* out, cudaStream_t st) {
    run(EPS_TC_SQNORM, 0.0, 4.0 * double(offsets[n] - offsets[0]), st, [&] {
      return eps_grad_sqnorm_flat(g32, offsets, n, out, act.sq_ws, act.sq_ws_bytes, st);
    });
  }

  void check_rows(int b0, int b) const {
    if (b0 < 0 || b < 1 || b0 + b > g.max_batch) throw int(EPS_EINVAL);
  }
  void check_span(int g0, int g1, int l_frozen) const {
    if (l_frozen < 0 || l_frozen >= g.layers || g0 < 0 || g1 < g0 || g1 > 2 * g.layers)
      throw int(EPS_EINVAL);
  }
};

namespace {

Geometry make_geom(const int* gi) {
  Geometry g{};
  g.layers = gi[0];
  g.d = gi[1];
  g.f = gi[2];
  g.heads = gi[3];
  g.tokens = gi[4];
  g.classes = gi[5];
  g.image = gi[6];
  g.in_image = gi[7];
  g.patch = gi[8];
  g.channels = gi[9];
  g.max_batch = gi[10];
  g.classes_pad = (g.classes + 7) / 8 * 8;
  if (g.layers < 1 || g.d % g.heads != 0 || g.tokens != g.patches() + 1 || g.max_batch < 1 ||
      g.classes < 1 || (g.d % 256 != 0 && g.d != 128))
    throw std::invalid_argument("vit geometry");
  return g;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return EPS_OK;
  } catch (int rc) {
    return rc;
  } catch (const std::bad_alloc&) {
    return EPS_ECAPACITY;
  } catch (...) {
    return EPS_EINVAL;
  }
}

}  // namespace

extern "C" {

// geom: {layers, d, mlp_dim, heads, tokens, classes, image, stored_image,
//        patch, channels, max_batch}.
// Outputs: param_total (elements of each fp32 / bf16 arena), workspace
// bytes, the L+1 layer segment offsets, and (optional) per-tensor offsets in
// the order: wpe bpe cls pos, per layer ln1g ln1b wqkv bqkv wp bp ln2g ln2b
// w1 b1 w2 b2, then lnfg lnfb wh bh  -> 4 + 12 L + 4 (offset, numel) pairs.
int eps_vit_layout(const int* geom, int64_t* param_total, int64_t* workspace_bytes,
                   int64_t* segments, int64_t* tensors) {
  return guard([&] {
    const Geometry g = make_geom(geom);
    const Layout lay(g);
    const Acts act(g, lay.total, nullptr);
    *param_total = lay.total;
    *workspace_bytes = int64_t(act.bytes);
    if (segments)
      for (size_t i = 0; i < lay.seg.size(); ++i) segments[i] = lay.seg[i];
    if (tensors) {
      int k = 0;
      auto put = [&](const Slot& s) {
        tensors[k++] = s.off;
        tensors[k++] = s.n;
      };
      put(lay.wpe), put(lay.bpe), put(lay.cls), put(lay.pos);
      for (const LayerSlots& s : lay.layer) {
        put(s.ln1g), put(s.ln1b), put(s.wqkv), put(s.bqkv), put(s.wp), put(s.bp);
        put(s.ln2g), put(s.ln2b), put(s.w1), put(s.b1), put(s.w2), put(s.b2);
      }
      put(lay.lnfg), put(lay.lnfb), put(lay.wh), put(lay.bh);
    }
  });
}

int eps_vit_create(const int* geom, float* params, uint16_t* params_bf16, float* grads,
                   float* momentum, void* workspace, eps_vit** out) {
  return guard([&] {
    *out = new eps_vit(make_geom(geom), params, params_bf16, grads, momentum,
                       static_cast<uint8_t*>(workspace));
  });
}

void eps_vit_destroy(eps_vit* h) { delete h; }

// One training iteration on a single stage holding the whole stack (K = 1):
// GPipe over `micro_batches` slices of the batch (integer split with the
// remainder on the leading slices, schedule.cpp:28-33): forward of every
// slice (head + loss + head backward right after each), then backward of
// every slice in reverse; grads accumulate in fp32.  Cache modes as in
// stage_fwd.  loss_sum (device fp32) accumulates the summed per-sample loss.
int eps_vit_train_step(eps_vit* h, const float* images, const int64_t* labels, int batch,
                       int micro_batches, int l_frozen, int cache_mode, int cache_old,
                       void* store, const int64_t* ids, float* loss_sum, void* stream) {
  return guard([&] {
    if (h == nullptr || batch < 1 || batch > h->g.max_batch || micro_batches < 1 ||
        micro_batches > batch || l_frozen < 0 || l_frozen >= h->g.layers)
      throw int(EPS_EINVAL);
    if (cache_mode != 0 && (store == nullptr || ids == nullptr || l_frozen == 0))
      throw int(EPS_EINVAL);
    if (cache_mode == 3 && (cache_old < 1 || cache_old >= l_frozen)) throw int(EPS_EINVAL);
    auto st = static_cast<cudaStream_t>(stream);
    h->loss_sum = loss_sum;
    const int g0 = 2 * l_frozen, g1 = 2 * h->g.layers;
    std::vector<int> b0s, bs;
    for (int m = 0, at = 0; m < micro_batches; ++m) {
      const int n = batch / micro_batches + (m < batch % micro_batches ? 1 : 0);
      b0s.push_back(at);
      bs.push_back(n);
      at += n;
    }
    for (int m = 0; m < micro_batches; ++m) {
      h->stage_fwd(images, b0s[m], bs[m], g0, g1, l_frozen, true, cache_mode, cache_old, store,
                   ids, st);
      h->head_fwd_bwd(labels, b0s[m], bs[m], batch, st);
    }
    for (int m = micro_batches - 1; m >= 0; --m)
      h->stage_bwd(b0s[m], bs[m], g0, g1, g0, l_frozen, false, st);
  });
}

// ---- pipeline stages (AutoPipe executor; host drives the GPipe order) ------
int eps_vit_stage_forward(eps_vit* h, const float* images, int b0, int b, int g0, int g1,
                          int l_frozen, int front, int cache_mode, int cache_old, void* store,
                          const int64_t* ids, void* stream) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->check_span(g0, g1, l_frozen);
    if (front && images == nullptr && cache_mode != 1) throw int(EPS_EINVAL);
    if (cache_mode != 0 &&
        (!front || store == nullptr || ids == nullptr || l_frozen == 0 || g0 < 2 * l_frozen))
      throw int(EPS_EINVAL);
    if (cache_mode == 3 && (cache_old < 1 || cache_old >= l_frozen)) throw int(EPS_EINVAL);
    h->stage_fwd(images, b0, b, g0, g1, l_frozen, front != 0, cache_mode, cache_old, store, ids,
                 static_cast<cudaStream_t>(stream));
  });
}

int eps_vit_stage_head(eps_vit* h, const int64_t* labels, int b0, int b, int global_batch,
                       float* loss_sum, void* stream) {
  return guard([&] {
    if (h == nullptr || labels == nullptr || loss_sum == nullptr || global_batch < 1)
      throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->loss_sum = loss_sum;
    h->head_fwd_bwd(labels, b0, b, global_batch, static_cast<cudaStream_t>(stream));
  });
}

int eps_vit_stage_backward(eps_vit* h, int b0, int b, int g0, int g1, int l_frozen,
                           int cut_out, void* stream) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->check_span(g0, g1, l_frozen);
    h->stage_bwd(b0, b, g0, g1, g0, l_frozen, cut_out != 0, static_cast<cudaStream_t>(stream));
  });
}

int eps_vit_stage_backward_part(eps_vit* h, int b0, int b, int g0, int g1, int stage_g0,
                                int l_frozen, int cut_out, void* stream) {
  return guard([&] {
    if (h == nullptr || stage_g0 > g0) throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->check_span(stage_g0, g1, l_frozen);
    h->stage_bwd(b0, b, g0, g1, stage_g0, l_frozen, cut_out != 0,
                 static_cast<cudaStream_t>(stream));
  });
}

// AutoCache store layout for cache_mode != 0: `table` (device uint64[n]) of
// shard base pointers with `rows_per_shard` sample rows each -- the store
// argument of the stage calls is then ignored except as a non-null marker;
// table = null reverts to a single store.
int eps_vit_set_cache_shards(eps_vit* h, const uint64_t* table, int64_t rows_per_shard) {
  return guard([&] {
    if (h == nullptr || (table != nullptr && rows_per_shard <= 0)) throw int(EPS_EINVAL);
    h->shard_table = table;
    h->rows_per_shard = table != nullptr ? rows_per_shard : 0;
  });
}

int eps_vit_set_redirect(eps_vit* h, int out_g, void* out_ptr, int dx_g, void* dx_ptr) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->out_g = out_g;
    h->out_to = static_cast<uint16_t*>(out_ptr);
    h->dx_g = dx_g;
    h->dx_to = static_cast<uint16_t*>(dx_ptr);
  });
}

void* eps_vit_cut(eps_vit* h, int g, int grad) {
  if (h == nullptr || g < 0 || g > 2 * h->g.layers) return nullptr;
  return grad ? static_cast<void*>(h->act.dX) : static_cast<void*>(h->cut(g));
}

int eps_vit_param_range(eps_vit* h, int g0, int g1, int64_t* begin, int64_t* end) {
  return guard([&] {
    if (h == nullptr || g0 < 0 || g1 < g0 || g1 > 2 * h->g.layers) throw int(EPS_EINVAL);
    *begin = h->sub_begin(g0);
    *end = h->sub_begin(g1);
  });
}

int eps_vit_sgd_range(eps_vit* h, int64_t begin, int64_t end, float lr, float momentum,
                      float weight_decay, void* stream) {
  return guard([&] {
    if (h == nullptr || begin < 0 || end > h->lay.total || end < begin) throw int(EPS_EINVAL);
    h->sgd_range(begin, end, lr, momentum, weight_decay, static_cast<cudaStream_t>(stream));
  });
}

int eps_vit_sqnorm_ranges(eps_vit* h, const int64_t* offsets, int n, double* out,
                          void* stream) {
  return guard([&] {
    if (h == nullptr || n < 1 || n > 64 || offsets[0] < 0 || offsets[n] > h->lay.total)
      throw int(EPS_EINVAL);
    h->sqnorm_ranges(offsets, n, out, static_cast<cudaStream_t>(stream));
  });
}

// Fused SGD-momentum over the trainable tail [segment L_f, end).
int eps_vit_sgd(eps_vit* h, int l_frozen, float lr, float momentum, float weight_decay,
                void* stream) {
  return guard([&] {
    h->sgd_range(h->lay.seg[l_frozen], h->lay.total, lr, momentum, weight_decay,
                 static_cast<cudaStream_t>(stream));
  });
}

// Per-layer gradient sum of squares (freeze test input) for layers
// [l_frozen, L) into out[l] (device double[L]); frozen layers are zeroed.
int eps_vit_layer_sqnorms(eps_vit* h, int l_frozen, double* out, void* stream) {
  return guard([&] {
    const int L = h->g.layers;
    auto st = static_cast<cudaStream_t>(stream);
    if (l_frozen > 0 && cudaMemsetAsync(out, 0, sizeof(double) * l_frozen, st) != cudaSuccess)
      throw int(EPS_ECUDA);
    std::vector<int64_t> offs(h->lay.seg.begin() + l_frozen, h->lay.seg.end());
    h->sqnorm_ranges(offs.data(), L - l_frozen, out + l_frozen, st);
  });
}

// Forward-only inference of the logits (used by tests): batch rows of
// images through all layers; logits bf16 [batch, classes_pad] into `logits`.
int eps_vit_forward_logits(eps_vit* h, const float* images, int batch, void* logits,
                           void* stream) {
  return guard([&] {
    auto st = static_cast<cudaStream_t>(stream);
    const int64_t d = h->g.d, T = h->g.tokens;
    h->check_rows(0, batch);
    h->embed_fwd(images, 0, batch, st);
    for (int l = 0; l < h->g.layers; ++l) {
      h->att_fwd(l, 0, batch, st);
      h->mlp_fwd(l, 0, batch, st);
    }
    const uint16_t* xl = h->act.X[h->g.layers];
    h->eltwise(st, [&] { return eps_gather_rows(xl, T * d, h->act.cls_rows, batch, d, 0, st); });
    h->layernorm(h->act.cls_rows, h->lay.lnfg, h->lay.lnfb, h->act.hf, h->act.meanf,
                 h->act.rstdf, batch, st);
    h->mm(0, 0, EPS_EPI_BIAS_BF16, h->act.hf, h->W(h->lay.wh), logits, h->P(h->lay.bh), nullptr,
          nullptr, batch, h->g.classes_pad, d, d, d, h->g.classes_pad, 1, st);
  });
}

// Device pointer to an internal activation buffer (tests / cache warm-up):
// which 0 = X[layer] (residual stream entering `layer`), 1 = dX scratch.
void* eps_vit_activation(eps_vit* h, int which, int layer) {
  if (which == 0 && layer >= 0 && layer <= h->g.layers) return h->act.X[layer];
  if (which == 1) return h->act.dX;
  return nullptr;
}

int eps_vit_set_side_stream(eps_vit* h, int on) {
  if (h == nullptr) return EPS_EINVAL;
  h->side_on = on != 0;
  return EPS_OK;
}

int eps_vit_timing_enable(eps_vit* h, int on) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->timing = on != 0;
    h->recs.clear();
    h->ev_used = 0;
  });
}

int eps_vit_timing_read(eps_vit* h, double* ms, double* flops, double* bytes, int64_t* count) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    for (int c = 0; c < EPS_TC_COUNT; ++c) {
      if (ms) ms[c] = 0;
      if (flops) flops[c] = 0;
      if (bytes) bytes[c] = 0;
      if (count) count[c] = 0;
    }
    for (const auto& r : h->recs) {
      if (cudaEventSynchronize(r.b) != cudaSuccess) throw int(EPS_ECUDA);
      float t = 0.f;
      if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) throw int(EPS_ECUDA);
      if (ms) ms[r.cls] += t;
      if (flops) flops[r.cls] += r.flops;
      if (bytes) bytes[r.cls] += r.bytes;
      if (count) count[r.cls] += 1;
    }
    h->recs.clear();
    h->ev_used = 0;
  });
}

}  // extern "C"
