// BERT training executor (BASELINE configs 4 and 5: BERT-base seq 384 with a
// SQuAD span head, BERT-large seq 128 with a pooled 2-class head).
//
// Same contract as the ViT executor (vit.cu): caller-owned parameter arenas
// in the reference's ModelSpec order (model.cpp:152-179: word / position /
// token-type embeddings + embedding LN folded into layer 0's ATT sublayer,
// pooler + classifier folded into layer L-1's MLP sublayer), caller-owned
// activation workspace, pipeline-stage operations over global sublayers
// [g0, g1) and the same freeze semantics.
//
// BERT is post-norm: ATT(x) = LN1(x + proj(attn(qkv(x)))),
// MLP(x1) = LN2(x1 + fc2(gelu(fc1(x1)))).  Every sublayer ends in its own
// LayerNorm, so every bias gradient is produced inside its sublayer's
// backward and stage cuts need no cross-stage column sums.
#include <cuda_runtime.h>

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
  Slot wqkv, bqkv, wp, bp, ln1g, ln1b;  // ATT sublayer (post-norm: LN1 last)
  Slot w1, b1, w2, b2, ln2g, ln2b;      // MLP sublayer
};

struct Geometry {
  int layers, d, f, heads, tokens, classes, vocab, positions, head_kind, pooler, max_batch;
  int classes_pad;
  int head_dim() const { return d / heads; }
};

constexpr int64_t kAlign = 64;

struct Layout {
  Slot word, pos, type, elng, elnb;
  std::vector<LayerSlots> layer;
  Slot wpool, bpool, wc, bc;
  std::vector<int64_t> seg;
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
    word = take(int64_t(g.vocab) * d);
    pos = take(int64_t(g.positions) * d);
    type = take(2 * d);
    elng = take(d);
    elnb = take(d);
    layer.resize(g.layers);
    for (int l = 0; l < g.layers; ++l) {
      if (l > 0) seg.push_back(at);
      LayerSlots& s = layer[l];
      s.wqkv = take(3 * d * d);
      s.bqkv = take(3 * d);
      s.wp = take(d * d);
      s.bp = take(d);
      s.ln1g = take(d);
      s.ln1b = take(d);
      s.w1 = take(f * d);
      s.b1 = take(f);
      s.w2 = take(d * f);
      s.b2 = take(d);
      s.ln2g = take(d);
      s.ln2b = take(d);
    }
    if (g.pooler) {
      wpool = take(d * d);
      bpool = take(d);
    }
    wc = take(int64_t(g.classes_pad) * d);
    bc = take(g.classes_pad);
    total = at;
    seg.push_back(total);
  }
};

struct Acts {
  uint16_t* E = nullptr;  // embedding sum (pre-LN)
  float *meanE = nullptr, *rstdE = nullptr;
  std::vector<uint16_t*> X, QKV, A, S1, X1, U, G, S2;
  std::vector<float*> mean1, rstd1, mean2, rstd2, lse;
  uint16_t *logits = nullptr, *dlogits = nullptr;               // QA: [R, cpad]
  uint16_t *cls = nullptr, *pre = nullptr, *pooled = nullptr;   // pooled head: [B, d]
  uint16_t *clog = nullptr, *dclog = nullptr, *dpooled = nullptr, *dpre = nullptr,
           *dcls = nullptr;
  uint16_t *dX = nullptr, *dS = nullptr, *dA = nullptr, *dQKV = nullptr;
  float* dsum = nullptr;
  float* drow = nullptr;  // attention D = rowsum(dO * O) [rows, heads] (ROWDOT epilogue)
  double* sq_ws = nullptr;
  size_t sq_ws_bytes = 0;
  size_t bytes = 0;

  Acts(const Geometry& g, int64_t param_total, uint8_t* base) {
    const int64_t B = g.max_batch, R = B * g.tokens, d = g.d, f = g.f, L = g.layers;
    const int64_t C = g.classes_pad;
    size_t at = 0;
    auto take = [&](size_t bytes) {
      uint8_t* p = base ? base + at : nullptr;
      at += (bytes + 255) / 256 * 256;
      return p;
    };
    auto bf = [&](int64_t n) { return reinterpret_cast<uint16_t*>(take(size_t(n) * 2)); };
    auto fp = [&](int64_t n) { return reinterpret_cast<float*>(take(size_t(n) * 4)); };
    E = bf(R * d);
    meanE = fp(R);
    rstdE = fp(R);
    for (int64_t l = 0; l <= L; ++l) X.push_back(bf(R * d));
    for (int64_t l = 0; l < L; ++l) {
      QKV.push_back(bf(R * 3 * d));
      A.push_back(bf(R * d));
      S1.push_back(bf(R * d));
      X1.push_back(bf(R * d));
      U.push_back(bf(R * f));
      G.push_back(bf(R * f));
      S2.push_back(bf(R * d));
      mean1.push_back(fp(R));
      rstd1.push_back(fp(R));
      mean2.push_back(fp(R));
      rstd2.push_back(fp(R));
      lse.push_back(fp(B * g.heads * g.tokens));
    }
    if (g.head_kind == 1) {
      logits = bf(R * C);
      dlogits = bf(R * C);
    } else {
      cls = bf(B * d);
      pre = bf(B * d);
      pooled = bf(B * d);
      clog = bf(B * C);
      dclog = bf(B * C);
      dpooled = bf(B * d);
      dpre = bf(B * d);
      dcls = bf(B * d);
    }
    dX = bf(R * d);
    dS = bf(R * d);
    dA = bf(R * d);
    dQKV = bf(R * 3 * d);
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

struct eps_bert {
  Geometry g;
  Layout lay;
  Acts act;
  float* p32;
  uint16_t* p16;
  float* g32;
  float* mom;
  float* loss_sum = nullptr;
  // Stage hand-off over peer memory (see the ViT executor).
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
  eps_bert(const Geometry& geom, float* p, uint16_t* pb, float* gr, float* m, uint8_t* ws)
      : g(geom), lay(geom), act(geom, lay.total, ws), p32(p), p16(pb), g32(gr), mom(m) {}
  ~eps_bert() {
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  }

  // ---- per-class launch timing (same scheme as the ViT executor) -------------
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
      return eps_layernorm_fwd(x, P(gam), P(bet), y, mean, rstd, rows, g.d, 1e-12f, st);
    });
  }
  // dx = LN'(dy); dgamma / dbeta accumulate; colsum_dx (optional) = bias grad
  // of the sublayer output that fed this LayerNorm.
  void layernorm_bwd(const uint16_t* dy, const uint16_t* x, const Slot& gam, const Slot& bet,
                     const float* mean, const float* rstd, uint16_t* dx, float* colsum_dx,
                     int64_t rows, cudaStream_t st) {
    run(EPS_TC_NORM, 0.0, 6.0 * double(rows) * g.d, st, [&] {
      return eps_layernorm_bwd(dy, x, P(gam), mean, rstd, nullptr, dx, Gr(gam), Gr(bet),
                               colsum_dx, rows, g.d, nullptr, st);
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
  int split_for(int64_t rows) const { return rows >= 16384 ? 8 : rows >= 4096 ? 4 : 1; }

  uint16_t* cut(int gs) const {
    if (gs >= 2 * g.layers) return act.X[g.layers];
    return (gs % 2 == 0) ? act.X[gs / 2] : act.X1[gs / 2];
  }
  int64_t sub_begin(int gs) const {
    if (gs >= 2 * g.layers) return lay.total;
    return (gs % 2 == 0) ? lay.seg[gs / 2] : lay.layer[gs / 2].w1.off;
  }

  // ---- forward -----------------------------------------------------------------
  void embed_fwd(const int64_t* tok, const int64_t* seg, int b0, int b, cudaStream_t st) {
    const int64_t d = g.d, T = g.tokens, r0 = int64_t(b0) * T, R = int64_t(b) * T;
    eltwise(st, [&] {
      return eps_bert_embed_fwd(tok + r0, seg + r0, P(lay.word), P(lay.pos), P(lay.type),
                                act.E + r0 * d, b, g.tokens, d, st);
    });
    layernorm(act.E + r0 * d, lay.elng, lay.elnb, act.X[0] + r0 * d, act.meanE + r0,
              act.rstdE + r0, R, st);
  }

  void att_fwd(int l, int b0, int b, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    mm(0, 0, EPS_EPI_BIAS_BF16, act.X[l] + r0 * d, W(s.wqkv), act.QKV[l] + r0 * 3 * d,
       P(s.bqkv), nullptr, nullptr, R, 3 * d, d, d, d, 3 * d, 1, st);
    const double t = g.tokens, hd = double(g.heads) * g.head_dim();
    run(EPS_TC_ATTN, 4.0 * b * t * t * hd, 8.0 * b * t * hd, st, [&] {
      return eps_attn_fwd(act.QKV[l] + r0 * 3 * d, act.A[l] + r0 * d,
                          act.lse[l] + int64_t(b0) * g.heads * g.tokens, b, g.tokens, g.heads,
                          g.head_dim(), scale(), st);
    });
    mm(0, 0, EPS_EPI_BIAS_RESID_BF16, act.A[l] + r0 * d, W(s.wp), act.S1[l] + r0 * d, P(s.bp),
       act.X[l] + r0 * d, nullptr, R, d, d, d, d, d, 1, st);
    layernorm(act.S1[l] + r0 * d, s.ln1g, s.ln1b, out_buf(2 * l + 1, act.X1[l]) + r0 * d,
              act.mean1[l] + r0, act.rstd1[l] + r0, R, st);
  }

  void mlp_fwd(int l, int b0, int b, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, f = g.f, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    mm(0, 0, EPS_EPI_BIAS_GELU2_BF16, act.X1[l] + r0 * d, W(s.w1), act.G[l] + r0 * f, P(s.b1),
       act.U[l] + r0 * f, nullptr, R, f, d, d, d, f, 1, st);
    mm(0, 0, EPS_EPI_BIAS_RESID_BF16, act.G[l] + r0 * f, W(s.w2), act.S2[l] + r0 * d, P(s.b2),
       act.X1[l] + r0 * d, nullptr, R, d, f, f, f, d, 1, st);
    layernorm(act.S2[l] + r0 * d, s.ln2g, s.ln2b, out_buf(2 * l + 2, act.X[l + 1]) + r0 * d,
              act.mean2[l] + r0, act.rstd2[l] + r0, R, st);
  }

  void sub_fwd(int gs, int b0, int b, cudaStream_t st) {
    if (gs % 2 == 0) att_fwd(gs / 2, b0, b, st);
    else mlp_fwd(gs / 2, b0, b, st);
  }

  // Head forward + loss + backward; leaves dL/dX[L] in the dX rows.
  //   head_kind 1 (SQuAD): per-token start/end logits, labels = [start[gb], end[gb]];
  //   head_kind 0: pooled CLS (tanh) -> classifier, labels = class[gb].
  void head_fwd_bwd(const int64_t* labels, int b0, int b, int global_batch, cudaStream_t st) {
    const int64_t d = g.d, C = g.classes_pad, T = g.tokens;
    const int64_t r0 = int64_t(b0) * T, R = int64_t(b) * T;
    uint16_t* xl = act.X[g.layers] + r0 * d;
    uint16_t* dX = act.dX + r0 * d;
    const float gs = 1.0f / float(global_batch);
    if (g.head_kind == 1) {
      uint16_t* lg = act.logits + r0 * C;
      uint16_t* dlg = act.dlogits + r0 * C;
      mm(0, 0, EPS_EPI_BIAS_BF16, xl, W(lay.wc), lg, P(lay.bc), nullptr, nullptr, R, C, d, d, d,
         C, 1, st);
      eltwise(st, [&] {
        return eps_span_xent(lg, labels + b0, labels + global_batch + b0, dlg, loss_sum,
                             Gr(lay.bc), b, g.tokens, int(C), gs, st);
      });
      mm(1, 1, EPS_EPI_ACCUM_F32, dlg, xl, Gr(lay.wc), nullptr, nullptr, nullptr, C, d, R, C, d, d,
         0, st);
      mm(0, 1, EPS_EPI_STORE_BF16, dlg, W(lay.wc), dX, nullptr, nullptr, nullptr, R, d, C, C, d, d,
         1, st);
      return;
    }
    uint16_t* cls = act.cls + int64_t(b0) * d;
    uint16_t* pre = act.pre + int64_t(b0) * d;
    uint16_t* pooled = act.pooled + int64_t(b0) * d;
    uint16_t* lg = act.clog + int64_t(b0) * C;
    uint16_t* dlg = act.dclog + int64_t(b0) * C;
    uint16_t* dpooled = act.dpooled + int64_t(b0) * d;
    uint16_t* dpre = act.dpre + int64_t(b0) * d;
    uint16_t* dcls = act.dcls + int64_t(b0) * d;
    eltwise(st, [&] { return eps_gather_rows(xl, T * d, cls, b, d, 0, st); });
    const uint16_t* feat = cls;
    if (g.pooler) {
      mm(0, 0, EPS_EPI_BIAS_BF16, cls, W(lay.wpool), pre, P(lay.bpool), nullptr, nullptr, b, d, d,
         d, d, d, 1, st);
      eltwise(st, [&] { return eps_tanh_fwd(pre, pooled, int64_t(b) * d, st); });
      feat = pooled;
    }
    mm(0, 0, EPS_EPI_BIAS_BF16, feat, W(lay.wc), lg, P(lay.bc), nullptr, nullptr, b, C, d, d, d, C,
       1, st);
    eltwise(st, [&] {
      return eps_softmax_xent_bias(lg, labels + b0, dlg, loss_sum, Gr(lay.bc), b, g.classes,
                                   int(C), gs, st);
    });
    mm(1, 1, EPS_EPI_ACCUM_F32, dlg, feat, Gr(lay.wc), nullptr, nullptr, nullptr, C, d, b, C, d, d,
       1, st);
    uint16_t* dfeat = g.pooler ? dpooled : dcls;
    mm(0, 1, EPS_EPI_STORE_BF16, dlg, W(lay.wc), dfeat, nullptr, nullptr, nullptr, b, d, C, C, d, d,
       1, st);
    if (g.pooler) {
      eltwise(st, [&] { return eps_tanh_bwd(dpooled, pooled, dpre, int64_t(b) * d, st); });
      eltwise(st, [&] { return eps_colsum_bf16(dpre, Gr(lay.bpool), b, d, st); });
      mm(1, 1, EPS_EPI_ACCUM_F32, dpre, cls, Gr(lay.wpool), nullptr, nullptr, nullptr, d, d, b, d,
         d, d, 1, st);
      mm(0, 1, EPS_EPI_STORE_BF16, dpre, W(lay.wpool), dcls, nullptr, nullptr, nullptr, b, d, d, d,
         d, d, 1, st);
    }
    if (cudaMemsetAsync(dX, 0, size_t(R) * d * 2, st) != cudaSuccess) throw int(EPS_ECUDA);
    eltwise(st, [&] { return eps_scatter_rows(dcls, dX, T * d, b, d, 0, st); });
  }

  // ---- backward ----------------------------------------------------------------
  void mlp_bwd(int l, int b0, int b, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, f = g.f, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    uint16_t* dX = act.dX + r0 * d;
    uint16_t* dS = act.dS + r0 * d;
    uint16_t* Gm = act.G[l] + r0 * f;
    const int split = 0;  // auto split-K (eps_gemm_bf16)
    layernorm_bwd(dX, act.S2[l] + r0 * d, s.ln2g, s.ln2b, act.mean2[l] + r0, act.rstd2[l] + r0, dS,
                  Gr(s.b2), R, st);
    mm(1, 1, EPS_EPI_ACCUM_F32, dS, Gm, Gr(s.w2), nullptr, nullptr, nullptr, d, f, R, d, f, f,
       split, st);
    mm(0, 1, EPS_EPI_MUL_BF16, dS, W(s.w2), Gm, nullptr, act.U[l] + r0 * f, Gr(s.b1), R, f, d, d,
       f, f, 1, st);
    mm(1, 1, EPS_EPI_ACCUM_F32, Gm, act.X1[l] + r0 * d, Gr(s.w1), nullptr, nullptr, nullptr, f, d,
       R, f, d, d, split, st);
    // dX1 = dU W1 + dS2 (the residual branch of the post-norm block)
    mm(0, 1, EPS_EPI_RESID_BF16, Gm, W(s.w1), dx_buf(2 * l + 1) + r0 * d, nullptr, dS, nullptr, R,
       d, f, f, d, d, 1, st);
  }

  void att_bwd(int l, int b0, int b, bool need_dx, cudaStream_t st) {
    const LayerSlots& s = lay.layer[l];
    const int64_t d = g.d, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    uint16_t* dX = act.dX + r0 * d;
    uint16_t* dS = act.dS + r0 * d;
    const int split = 0;  // auto split-K (eps_gemm_bf16)
    layernorm_bwd(dX, act.S1[l] + r0 * d, s.ln1g, s.ln1b, act.mean1[l] + r0, act.rstd1[l] + r0, dS,
                  Gr(s.bp), R, st);
    mm(1, 1, EPS_EPI_ACCUM_F32, dS, act.A[l] + r0 * d, Gr(s.wp), nullptr, nullptr, nullptr, d, d,
       R, d, d, d, split, st);
    // dA = dX1 W_o; for the fused attention backward its epilogue also forms
    // D = rowsum(dA * A) per (row, head) (EPS_EPI_ROWDOT_BF16)
    const bool rowdot = eps_attn_bwd_uses_rowdot(g.tokens, g.head_dim()) != 0;
    float* drow = act.drow + r0 * g.heads;
    if (rowdot) cudaMemsetAsync(drow, 0, size_t(R) * g.heads * sizeof(float), st);
    mm(0, 1, rowdot ? EPS_EPI_ROWDOT_BF16 : EPS_EPI_STORE_BF16, dS, W(s.wp), act.dA + r0 * d,
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
    mm(1, 1, EPS_EPI_ACCUM_F32, act.dQKV + r0 * 3 * d, act.X[l] + r0 * d, Gr(s.wqkv), nullptr,
       nullptr, nullptr, 3 * d, d, R, 3 * d, d, d, split, st);
    if (need_dx)  // dX = dQKV Wqkv + dS1
      mm(0, 1, EPS_EPI_RESID_BF16, act.dQKV + r0 * 3 * d, W(s.wqkv), dx_buf(2 * l) + r0 * d,
         nullptr, dS, nullptr, R, d, 3 * d, 3 * d, d, d, 1, st);
  }

  void embed_bwd(const int64_t* tok, const int64_t* seg, int b0, int b, cudaStream_t st) {
    const int64_t d = g.d, r0 = int64_t(b0) * g.tokens, R = int64_t(b) * g.tokens;
    uint16_t* dS = act.dS + r0 * d;
    layernorm_bwd(act.dX + r0 * d, act.E + r0 * d, lay.elng, lay.elnb, act.meanE + r0,
                  act.rstdE + r0, dS, nullptr, R, st);
    eltwise(st, [&] {
      return eps_bert_embed_bwd(dS, tok + r0, seg + r0, Gr(lay.word), Gr(lay.pos), Gr(lay.type), b,
                                g.tokens, d, st);
    });
  }

  // ---- stages --------------------------------------------------------------------
  // inputs: tokens [B*T] int64 followed by segment ids [B*T] (front stage).
  const int64_t* tok_in = nullptr;
  const int64_t* seg_in = nullptr;

  void stage_fwd(const int64_t* inputs, int batch_rows, int b0, int b, int g0, int g1,
                 int l_frozen, bool front, int cache_mode, int cache_old, void* store,
                 const int64_t* ids, cudaStream_t st) {
    const int64_t xoff = int64_t(b0) * g.tokens * g.d;
    const int64_t rb = int64_t(g.tokens) * g.d * 2;
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
      if (inputs != nullptr) {
        tok_in = inputs;
        seg_in = inputs + int64_t(batch_rows) * g.tokens;
      }
      int start = 0;
      if (cache_mode == 1) {
        cache_io(true, act.X[l_frozen]);
        start = l_frozen;
      } else if ((cache_mode == 2 || cache_mode == 3) && cache_old > 0) {
        cache_io(true, act.X[cache_old]);
        start = cache_old;
      }
      if (start == 0 && cache_mode != 1) embed_fwd(tok_in, seg_in, b0, b, st);
      for (int l = start; l < l_frozen; ++l) {
        att_fwd(l, b0, b, st);
        mlp_fwd(l, b0, b, st);
      }
      if (cache_mode == 2) cache_io(false, act.X[l_frozen]);
    }
    for (int gs = g0; gs < g1; ++gs) sub_fwd(gs, b0, b, st);
  }

  void stage_bwd(int b0, int b, int g0, int g1, int l_frozen, cudaStream_t st) {
    if (g1 <= g0) return;
    for (int gs = g1 - 1; gs >= g0; --gs) {
      const int l = gs / 2;
      if (gs % 2 == 1) mlp_bwd(l, b0, b, st);
      else att_bwd(l, b0, b, l > l_frozen || l == 0, st);
    }
    if (g0 == 0 && l_frozen == 0) embed_bwd(tok_in, seg_in, b0, b, st);
  }

  void sgd_range(int64_t begin, int64_t end, float lr, float mu, float wd, cudaStream_t st) {
    if (end <= begin) return;
    run(EPS_TC_OPTIM, 0.0, 26.0 * double(end - begin), st, [&] {
      return eps_sgd_momentum(p32 + begin, p16 + begin, g32 + begin, mom + begin, end - begin, lr,
                              mu, wd, st);
    });
  }
  void adamw_range(int64_t begin, int64_t end, float lr, float b1, float b2, float eps, float wd,
                   int step, cudaStream_t st) {
    if (end <= begin) return;
    // AdamW keeps m in `mom` and v in the second half of the caller's state
    run(EPS_TC_OPTIM, 0.0, 34.0 * double(end - begin), st, [&] {
      return eps_adamw(p32 + begin, p16 + begin, g32 + begin, mom + begin,
                       mom + lay.total + begin, end - begin, lr, b1, b2, eps, wd, step, st);
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
    if (l_frozen < 0 || l_frozen >= g.layers || g0 < 2 * l_frozen || g1 < g0 ||
        g1 > 2 * g.layers)
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
  g.vocab = gi[6];
  g.positions = gi[7];
  g.head_kind = gi[8];
  g.pooler = gi[9];
  g.max_batch = gi[10];
  g.classes_pad = (g.classes + 7) / 8 * 8;
  if (g.layers < 1 || g.d % g.heads != 0 || g.tokens < 1 || g.tokens > g.positions ||
      g.max_batch < 1 || g.classes < 1 || g.vocab < 1 || (g.head_kind == 1 && g.classes != 2) ||
      (g.d % 256 != 0 && g.d != 128))
    throw std::invalid_argument("bert geometry");
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

// geom: {layers, d, mlp_dim, heads, tokens, classes, vocab, positions,
//        head_kind (0 pooled-CLS classifier, 1 SQuAD span), pooler, max_batch}.
// tensors (optional): (offset, numel) pairs in the order word pos type elng
// elnb, per layer wqkv bqkv wp bp ln1g ln1b w1 b1 w2 b2 ln2g ln2b, then
// [wpool bpool] wc bc.
int eps_bert_layout(const int* geom, int64_t* param_total, int64_t* workspace_bytes,
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
      put(lay.word), put(lay.pos), put(lay.type), put(lay.elng), put(lay.elnb);
      for (const LayerSlots& s : lay.layer) {
        put(s.wqkv), put(s.bqkv), put(s.wp), put(s.bp), put(s.ln1g), put(s.ln1b);
        put(s.w1), put(s.b1), put(s.w2), put(s.b2), put(s.ln2g), put(s.ln2b);
      }
      if (g.pooler) put(lay.wpool), put(lay.bpool);
      put(lay.wc), put(lay.bc);
    }
  });
}

int eps_bert_create(const int* geom, float* params, uint16_t* params_bf16, float* grads,
                    float* state, void* workspace, eps_bert** out) {
  return guard([&] {
    *out = new eps_bert(make_geom(geom), params, params_bf16, grads, state,
                        static_cast<uint8_t*>(workspace));
  });
}

void eps_bert_destroy(eps_bert* h) { delete h; }

int eps_bert_stage_forward(eps_bert* h, const int64_t* inputs, int batch_rows, int b0, int b,
                           int g0, int g1, int l_frozen, int front, int cache_mode, int cache_old,
                           void* store, const int64_t* ids, void* stream) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->check_span(g0, g1, l_frozen);
    if (front && inputs == nullptr && cache_mode != 1 && h->tok_in == nullptr)
      throw int(EPS_EINVAL);
    if (cache_mode != 0 && (!front || store == nullptr || ids == nullptr || l_frozen == 0))
      throw int(EPS_EINVAL);
    if (cache_mode == 3 && (cache_old < 1 || cache_old >= l_frozen))
      throw int(EPS_EINVAL);
    h->stage_fwd(inputs, batch_rows, b0, b, g0, g1, l_frozen, front != 0, cache_mode, cache_old,
                 store, ids, static_cast<cudaStream_t>(stream));
  });
}

int eps_bert_stage_head(eps_bert* h, const int64_t* labels, int b0, int b, int global_batch,
                        float* loss_sum, void* stream) {
  return guard([&] {
    if (h == nullptr || labels == nullptr || loss_sum == nullptr || global_batch < 1)
      throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->loss_sum = loss_sum;
    h->head_fwd_bwd(labels, b0, b, global_batch, static_cast<cudaStream_t>(stream));
  });
}

int eps_bert_stage_backward_part(eps_bert* h, int b0, int b, int g0, int g1, int stage_g0,
                                 int l_frozen, int cut_out, void* stream) {
  (void)cut_out;
  (void)stage_g0;  // post-norm: every bias gradient stays inside its sublayer
  return guard([&] {
    if (h == nullptr || stage_g0 > g0) throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->check_span(g0, g1, l_frozen);
    h->stage_bwd(b0, b, g0, g1, l_frozen, static_cast<cudaStream_t>(stream));
  });
}

int eps_bert_stage_backward(eps_bert* h, int b0, int b, int g0, int g1, int l_frozen,
                            int cut_out, void* stream) {
  (void)cut_out;  // post-norm: bias grads never straddle a cut
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->check_rows(b0, b);
    h->check_span(g0, g1, l_frozen);
    h->stage_bwd(b0, b, g0, g1, l_frozen, static_cast<cudaStream_t>(stream));
  });
}

// AutoCache store layout for cache_mode != 0: `table` (device uint64[n]) of
// shard base pointers with `rows_per_shard` sample rows each -- the store
// argument of the stage calls is then ignored except as a non-null marker;
// table = null reverts to a single store.
int eps_bert_set_cache_shards(eps_bert* h, const uint64_t* table, int64_t rows_per_shard) {
  return guard([&] {
    if (h == nullptr || (table != nullptr && rows_per_shard <= 0)) throw int(EPS_EINVAL);
    h->shard_table = table;
    h->rows_per_shard = table != nullptr ? rows_per_shard : 0;
  });
}

int eps_bert_set_redirect(eps_bert* h, int out_g, void* out_ptr, int dx_g, void* dx_ptr) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->out_g = out_g;
    h->out_to = static_cast<uint16_t*>(out_ptr);
    h->dx_g = dx_g;
    h->dx_to = static_cast<uint16_t*>(dx_ptr);
  });
}

void* eps_bert_cut(eps_bert* h, int g, int grad) {
  if (h == nullptr || g < 0 || g > 2 * h->g.layers) return nullptr;
  return grad ? static_cast<void*>(h->act.dX) : static_cast<void*>(h->cut(g));
}

int eps_bert_param_range(eps_bert* h, int g0, int g1, int64_t* begin, int64_t* end) {
  return guard([&] {
    if (h == nullptr || g0 < 0 || g1 < g0 || g1 > 2 * h->g.layers) throw int(EPS_EINVAL);
    *begin = h->sub_begin(g0);
    *end = h->sub_begin(g1);
  });
}

int eps_bert_sgd_range(eps_bert* h, int64_t begin, int64_t end, float lr, float momentum,
                       float weight_decay, void* stream) {
  return guard([&] {
    if (h == nullptr || begin < 0 || end > h->lay.total || end < begin) throw int(EPS_EINVAL);
    h->sgd_range(begin, end, lr, momentum, weight_decay, static_cast<cudaStream_t>(stream));
  });
}

int eps_bert_adamw_range(eps_bert* h, int64_t begin, int64_t end, float lr, float beta1,
                         float beta2, float eps, float weight_decay, int step, void* stream) {
  return guard([&] {
    if (h == nullptr || begin < 0 || end > h->lay.total || end < begin || step < 1)
      throw int(EPS_EINVAL);
    h->adamw_range(begin, end, lr, beta1, beta2, eps, weight_decay, step,
                   static_cast<cudaStream_t>(stream));
  });
}

int eps_bert_sqnorm_ranges(eps_bert* h, const int64_t* offsets, int n, double* out,
                           void* stream) {
  return guard([&] {
    if (h == nullptr || n < 1 || n > 64 || offsets[0] < 0 || offsets[n] > h->lay.total)
      throw int(EPS_EINVAL);
    h->sqnorm_ranges(offsets, n, out, static_cast<cudaStream_t>(stream));
  });
}

int eps_bert_timing_enable(eps_bert* h, int on) {
  return guard([&] {
    if (h == nullptr) throw int(EPS_EINVAL);
    h->timing = on != 0;
    h->recs.clear();
    h->ev_used = 0;
  });
}

int eps_bert_timing_read(eps_bert* h, double* ms, double* flops, double* bytes, int64_t* count) {
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
