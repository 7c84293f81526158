// The device engine: allocation and geometry (shards, column windows, capacity),
// per-chunk launch plans, host->device uploads, and the builds (device-resident,
// streamed from host buffers, k-point batches).  The collective and the downloads are
// in reduce.cpp.
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>

#include "device.hpp"
#include "engine.hpp"
#include "host_pool.hpp"

namespace hsdla_b200 {

void check_dims(uint64_t na, uint64_t nl, uint64_t ng) {
  if (na < 1 || nl < 1 || ng < 1) throw Fail{HSDLA_B200_DIMENSION_ERROR, "all dims must be >= 1"};
  const uint64_t max = UINT64_MAX / 16 / 4;
  if (na > max / nl) throw Fail{HSDLA_B200_SIZING_ERROR, "n_atoms * n_l overflows"};
  if (na * nl > max / ng) throw Fail{HSDLA_B200_SIZING_ERROR, "problem allocation overflows"};
  if (ng > (1u << 31) - 1 || na * nl > (1u << 30) || nl > 4096)
    throw Fail{HSDLA_B200_SIZING_ERROR, "dimension exceeds the supported coordinate range"};
}

bool valid_algo(int algo) {
  return algo == HSDLA_B200_ALGO_REFINED || algo == HSDLA_B200_ALGO_REFINED_FUSED ||
         algo == HSDLA_B200_ALGO_REFINED_MERGED || algo == HSDLA_B200_ALGO_ORIGINAL;
}

template <class T>
static void dalloc(hsdla_b200_engine* e, T** p, uint64_t count) {
  const uint64_t bytes = std::max<uint64_t>(count * sizeof(T), 16);
  HS_CUDA(cudaMalloc(reinterpret_cast<void**>(p), bytes));
  e->device_bytes += bytes;
}

void engine_free(hsdla_b200_engine* e) {
  cudaSetDevice(e->device);
  // nothing of this engine may still be in flight
  for (cudaStream_t s : {e->stream, e->copy_stream, e->comm_stream, e->h2d_stream})
    if (s) cudaStreamSynchronize(s);
  for (void* p : {e->lapw_scratch, (void*)e->info, (void*)e->n_fail, (void*)e->sk_ws, (void*)e->sk_flags,
                  (void*)e->Aset[0], (void*)e->Bset[0], (void*)e->Aset[1], (void*)e->Bset[1], (void*)e->X1,
                  (void*)e->X2, (void*)e->Tab, (void*)e->Taa, (void*)e->Tbb, (void*)e->Paa, (void*)e->Pbb,
                  (void*)e->Wl, (void*)e->U, (void*)e->Hp, (void*)e->Sp, (void*)e->d_stamp})
    if (p) cudaFree(p);
  if (e->host_stage) cudaFreeHost(e->host_stage);
  for (double2* st : e->host_stage_x)
    if (st) cudaFreeHost(st);
  release_file_view(e);
  for (cudaEvent_t ev : {e->ev_kup[0], e->ev_kup[1], e->ev_kbuilt[0], e->ev_kbuilt[1]})
    if (ev) cudaEventDestroy(ev);
  if (e->h2d_stream) cudaStreamDestroy(e->h2d_stream);
  for (int i = 0; i < hsdla_b200_engine::kStageSlabs; ++i) {
    if (e->stage_ev[i]) cudaEventDestroy(e->stage_ev[i]);
    if (e->stage_buf[i]) cudaFreeHost(e->stage_buf[i]);
  }
  for (cudaEvent_t ev : e->tr_pool) cudaEventDestroy(ev);
  for (cudaEvent_t ev : e->ev_chunk_up) cudaEventDestroy(ev);
  for (int q = 0; q < hsdla_b200_engine::kD2hPieces; ++q)
    for (cudaEvent_t ev : {e->ev_h_band[q], e->ev_h_red[q], e->ev_dl_h[q], e->ev_dlx_h[0][q], e->ev_dlx_h[1][q]})
      if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : {e->ev_a0, e->ev_ops, e->ev_cs_order, e->ev_begin, e->ev_end, e->ev_end_t, e->ev_s_done, e->ev_s_red, e->ev_reduce_end,
                         e->ev_up0, e->ev_up1, e->ev_dl_s, e->ev_dlx_s[0], e->ev_dlx_s[1], e->ev_setup0, e->ev_setup1, e->ev_setup_mid})
    if (ev) cudaEventDestroy(ev);
  for (auto& t : e->ring)
    for (cudaEvent_t ev : {t.s0, t.s1, t.h0, t.h1})
      if (ev) cudaEventDestroy(ev);
  if (e->comm && e->comm_owned) ncclCommDestroy(e->comm);
  for (cudaStream_t s : {e->stream, e->copy_stream, e->comm_stream})
    if (s) cudaStreamDestroy(s);
}

// ---- geometry ----------------------------------------------------------------------
static uint64_t tiles_of(uint64_t n) { return (n + kTriBM - 1) / kTriBM; }

// Lower tiles of the engine's window: all t(t+1)/2, or for tile columns [t0, t1) the
// triangle of rows t0..t1-1 plus the full-width rows t1..T-1 (ctn_contract.cuh tri_tile_strict
// enumerates the strictly-lower ones, the diagonal tiles run in a launch of their own).
static uint64_t window_tiles(uint64_t T, uint64_t t0, uint64_t t1) {
  const uint64_t w = t1 - t0;
  return w * (w + 1) / 2 + (T - t1) * w;
}

static bool whole(const hsdla_b200_engine* e) { return e->c0 == 0 && e->c1 == e->ng; }

static void check_window(uint64_t ng, uint64_t c0, uint64_t c1) {
  if (c0 % kTriBM != 0 || c0 >= c1 || c1 > ng || (c1 != ng && c1 % kTriBM != 0))
    throw Fail{HSDLA_B200_CONFIG_ERROR,
               "column window [c0, c1) must satisfy c0 < c1 <= n_g, with c0 and c1 (unless n_g) multiples of 64"};
}

static void set_seg(CtnParams& P, int s, const CUtensorMap& L, const CUtensorMap& R, uint64_t Kc) {
  P.L[s] = L;
  P.R[s] = R;
  P.kchunks[s] = chunks_of(Kc);
  P.l_row_z[s] = 0;
  P.r_row_z[s] = 0;
}

// Parameter blocks for atoms [a0, a1) of A/B set `set`.  `first` = the chunk that starts
// H and S (beta 0); later chunks accumulate (beta 1).
static void make_chunk(hsdla_b200_engine* e, int set, uint64_t a0, uint64_t a1, bool first, ChunkPlan& cp) {
  const uint64_t K = e->K, ncol = e->ncol, nl = e->nl;
  const uint64_t r0 = a0 * nl, nac = a1 - a0;
  cp.a0 = a0;
  cp.a1 = a1;
  cp.A = e->A(set);
  cp.B = e->B(set);
  // the contractions sum over this chunk's rows inside the engine's row range [row0, row1)
  // (every atom of an engine touches the range, so tr1 > tr0)
  const uint64_t tr0 = std::max(r0, e->row0), tr1 = std::min(a1 * nl, e->row1), Kc = tr1 - tr0;
  if (tr1 <= tr0) throw Fail{HSDLA_B200_CONFIG_ERROR, "chunk outside the engine's row range"};
  // K-stacked buffers restricted to rows [tr0, tr1): {2Kc, ncol, 1}, column stride 2K
  // X2 is allocated on first use by the fused / original algorithms (the refined
  // algorithm needs X1 only); until then its maps alias X1 and are never launched.
  double2* x2 = e->X2 ? e->X2 : e->X1;
  CUtensorMap mA, mB, mX1, mX2;
  make_map(&mA, e->A(set) + tr0, 2 * Kc, ncol, 1, 2 * K, 2 * K * ncol, kTriBM, 1);
  make_map(&mB, e->B(set) + tr0, 2 * Kc, ncol, 1, 2 * K, 2 * K * ncol, kTriBM, 1);
  make_map(&mX1, e->X1 + tr0, 2 * Kc, ncol, 1, 2 * K, 2 * K * ncol, kTriBM, 1);
  make_map(&mX2, x2 + tr0, 2 * Kc, ncol, 1, 2 * K, 2 * K * ncol, kTriBM, 1);
  const uint64_t T = tiles_of(e->ng);
  const bool all = whole(e);
  const uint64_t t0 = e->c0 / kTriBM, t1 = tiles_of(e->c1);
  const uint64_t tri_tiles = all ? T * (T + 1) / 2 : window_tiles(T, t0, t1);
  if (tri_tiles > static_cast<uint64_t>(INT32_MAX)) throw Fail{HSDLA_B200_SIZING_ERROR, "too many lower tiles"};
  const double beta0 = first ? 0.0 : 1.0;
  auto tri_base = [&](CtnParams& P, double2* out, double beta) {
    std::memset(&P, 0, sizeof(P));
    P.n = static_cast<int>(e->ng);
    P.tiles = static_cast<int>(T);
    P.tiles_total = static_cast<int>(tri_tiles);
    if (!all) {  // the window's tile columns (tri_tile_strict order)
      P.col_t0 = static_cast<int>(t0);
      P.col_t1 = static_cast<int>(t1);
    }
    P.g0 = static_cast<int>(e->c0);
    P.pk0 = e->pk0;
    P.band = tri_band();
    P.out = out;
    P.sk_ws = e->sk_ws;
    P.sk_flags = e->sk_flags;
    P.alpha_re = 1.0;
    P.alpha_im = 0.0;
    P.beta = beta;
  };
  // phase s: S = A^H A + (U B)^H (U B)   (pipeline.cpp:298-300)
  tri_base(cp.s, e->Sp, beta0);
  set_seg(cp.s, 0, mA, mA, Kc);
  set_seg(cp.s, 1, mX1, mX1, Kc);
  cp.s.nseg = 2;
  tri_base(cp.sA, e->Sp, beta0);
  set_seg(cp.sA, 0, mA, mA, Kc);
  cp.sA.nseg = 1;
  tri_base(cp.sB, e->Sp, 1.0);
  set_seg(cp.sB, 0, mX1, mX1, Kc);
  cp.sB.nseg = 1;
  // fused H = Z^H B + B^H Z + A^H X   (pipeline.cpp:311 + :324)
  tri_base(cp.h, e->Hp, beta0);
  set_seg(cp.h, 0, mX2, mB, Kc);
  set_seg(cp.h, 1, mB, mX2, Kc);
  set_seg(cp.h, 2, mA, mX1, Kc);
  cp.h.nseg = 3;
  // reference-order her2k over Z in X1 (beta 0 on the first chunk) and herkx (always accumulates)
  tri_base(cp.h2k, e->Hp, beta0);
  set_seg(cp.h2k, 0, mX1, mB, Kc);
  set_seg(cp.h2k, 1, mB, mX1, Kc);
  cp.h2k.nseg = 2;
  tri_base(cp.hkx, e->Hp, 1.0);
  set_seg(cp.hkx, 0, mA, mX1, Kc);
  cp.hkx.nseg = 1;
  // merged H = A^H W_A + B^H W_B (W_A in X1, W_B in X2)
  tri_base(cp.hm, e->Hp, beta0);
  set_seg(cp.hm, 0, mA, mX1, Kc);
  set_seg(cp.hm, 1, mB, mX2, Kc);
  cp.hm.nseg = 2;
  // original h_aa_update: H += Lft^H W (Lft in X2, W = Q^H A in X1), always accumulates
  tri_base(cp.haa, e->Hp, 1.0);
  set_seg(cp.haa, 0, mX2, mX1, Kc);
  cp.haa.nseg = 1;
  cp.haa.keep_diag_imag = e->n_fail;  // keep the fold's diagonal imaginary part once an atom failed
  // persistent stream-K grid: one CTA per SM, never more CTAs than k-iterations
  cp.grid_tri = dim3(static_cast<unsigned>(std::min<uint64_t>(e->sms, tri_tiles * chunks_of(Kc))));

  // batched per-atom products over the held columns: operators {2nl, nl, nac} (row i in
  // dim 1, atom in dim 2), coefficient views {2nl, nac, ncol} (atom in dim 1, G in dim 2).
  const uint64_t blk = nl * nl;
  CUtensorMap mTab, mPbb, mPaa, mW0, mW1, vA, vB;
  make_map(&mTab, e->Tab + a0 * blk, 2 * nl, nl, nac, 2 * nl, 2 * blk, kBatBM, 1);
  make_map(&mPbb, e->Pbb + a0 * blk, 2 * nl, nl, nac, 2 * nl, 2 * blk, kBatBM, 1);
  make_map(&mPaa, e->Paa + a0 * blk, 2 * nl, nl, nac, 2 * nl, 2 * blk, kBatBM, 1);
  // merged: the stacked left operand {2nl (k), 2nl (output row), nac}, atom stride 4 blk
  make_map(&mW0, e->Wl + 4 * a0 * blk, 2 * nl, 2 * nl, nac, 2 * nl, 8 * blk, kBatWBM, 1);
  make_map(&mW1, e->Wl + 4 * a0 * blk + 2 * blk, 2 * nl, 2 * nl, nac, 2 * nl, 8 * blk, kBatWBM, 1);
  make_map(&vA, e->A(set) + r0, 2 * nl, nac, ncol, 2 * nl, 2 * K, 1, kBatBN);
  make_map(&vB, e->B(set) + r0, 2 * nl, nac, ncol, 2 * nl, 2 * K, 1, kBatBN);
  // the W launch's tile width: 192 columns (wider warp tiles: 1.15 against 1.18 ms at C2) unless
  // 128 pads N_G less (N_G 1000: 1024 against 1152 columns)
  const uint64_t pad192 = (ncol + kBatWBN - 1) / kBatWBN * kBatWBN, pad128 = (ncol + kBatBN - 1) / kBatBN * kBatBN;
  cp.w_bn = pad192 <= pad128 + ncol / 64 ? kBatWBN : kBatBN;
  CUtensorMap wA, wB;
  make_map(&wA, e->A(set) + r0, 2 * nl, nac, ncol, 2 * nl, 2 * K, 1, cp.w_bn);
  make_map(&wB, e->B(set) + r0, 2 * nl, nac, ncol, 2 * nl, 2 * K, 1, cp.w_bn);
  const int bat_tx = static_cast<int>((ncol + kBatBN - 1) / kBatBN), bat_ty = static_cast<int>((nl + kBatBM - 1) / kBatBM);
  const uint64_t bat_tiles = static_cast<uint64_t>(bat_tx) * bat_ty * nac;
  const int batw_ty = static_cast<int>((2 * nl + kBatWBM - 1) / kBatWBM);
  const int batw_tx = static_cast<int>((ncol + cp.w_bn - 1) / cp.w_bn);
  const uint64_t batw_tiles = static_cast<uint64_t>(batw_tx) * batw_ty * nac;
  if (batw_tiles > static_cast<uint64_t>(INT32_MAX)) throw Fail{HSDLA_B200_SIZING_ERROR, "too many batched tiles"};
  // N_L mod 8 in [1, 4]: each segment's last k-slab is half zero-fill (skipped by the kernel)
  const int half = nl % kChunkC >= 1 && nl % kChunkC <= kChunkC / 2;
  auto bat_base = [&](CtnParams& P, double2* out) {
    std::memset(&P, 0, sizeof(P));
    P.n = static_cast<int>(ncol);
    P.m_valid = static_cast<int>(nl);
    P.out = out;
    P.ldo = K;
    P.alpha_re = 1.0;
    P.bat_tx = bat_tx;
    P.bat_ty = bat_ty;
    P.bat_tiles = static_cast<int>(bat_tiles);
  };
  // Z_a = T_AB^H A_a + (1/2 T_BB) B_a   (compute_z, pipeline.cpp:176-185): into X1
  // (refined / original) or X2 (fused, where X1 still holds T_AA A for the same launch)
  bat_base(cp.z, e->X1 + r0);
  cp.z.L[0] = mTab;
  cp.z.R[0] = vA;
  cp.z.L[1] = mPbb;
  cp.z.R[1] = vB;
  cp.z.kchunks[0] = cp.z.kchunks[1] = chunks_of(nl);
  cp.z.half_last[0] = cp.z.half_last[1] = half;
  cp.z.r_row_z[0] = cp.z.r_row_z[1] = 1;
  cp.z.nseg = 2;
  cp.zf = cp.z;
  cp.zf.out = x2 + r0;
  // X_a = T_AA A_a (hemm_loop, pipeline.cpp:314-321); in the original algorithm Paa
  // holds the potrf output Q_a, so the same launch is trmm(L^H) / hemm per atom
  bat_base(cp.x, e->X1 + r0);
  cp.x.L[0] = mPaa;
  cp.x.R[0] = vA;
  cp.x.kchunks[0] = chunks_of(nl);
  cp.x.half_last[0] = half;
  cp.x.r_row_z[0] = 1;
  cp.x.nseg = 1;
  // merged: [W_A; W_B] = M_a [A_a; B_a] in ONE launch over 2 N_L output rows per atom:
  // segment 0 (k over A_a) reads [Paa | Tab], segment 1 (k over B_a) [Pab | Pbb];
  // rows < N_L (W_A) go to X1, the rest (W_B) to X2
  bat_base(cp.w, e->X1 + r0);
  cp.w.L[0] = mW0;
  cp.w.R[0] = wA;
  cp.w.L[1] = mW1;
  cp.w.R[1] = wB;
  cp.w.kchunks[0] = cp.w.kchunks[1] = chunks_of(nl);
  cp.w.half_last[0] = cp.w.half_last[1] = half;
  cp.w.r_row_z[0] = cp.w.r_row_z[1] = 1;
  cp.w.nseg = 2;
  cp.w.m_valid = static_cast<int>(2 * nl);
  cp.w.m_row = static_cast<int>(nl);
  cp.w.out2 = x2 + r0;
  cp.w.bat_tx = batw_tx;
  cp.w.bat_ty = batw_ty;
  cp.w.bat_tiles = static_cast<int>(batw_tiles);
  cp.grid_batw = dim3(static_cast<unsigned>(std::min<uint64_t>(batw_tiles, e->sms)));
  // persistent: one CTA per SM (the 384-thread CTA holds the whole register file)
  cp.grid_bat = dim3(static_cast<unsigned>(std::min<uint64_t>(bat_tiles, e->sms)));
}

// Streamed chunking for the host-buffer drop-in: whole-atom chunks, chunk c+1's upload
// overlapping chunk c's phases.  The plan minimises a model of the call's device timeline by
// dynamic programming over the chunk boundaries (at most 8 chunks):
//   chunk k of s_k atoms starts at max(end of chunk k-1, its upload done = u x atoms so far)
//   and takes c x s_k + f,
// with u = one atom's A and B rows at `rate` (host -> device feed: ~50 GB/s page-locked, ~35
// GB/s effective for rows the host packs into pinned slabs or copies from the page cache),
// c = one atom's share of the executed flops (merged 3M: S and H over the window's tiles, W)
// at 33 TF/s, and f = a chunk's fixed cost (launch ramps and tails, the beta = 1 passes over the
// packed H, S: 50 us + the window's packed bytes x 4 at 2 TB/s; ~0.2 ms at C2).  C2 pinned: the
// plan 2,4,9,17,32 atoms ran 19.9 ms per call against 20.2 for the earlier geometric plan
// 4,9,20,31 (tools/small_probe.py).  Small problems (< 4M A elements) stay one chunk: there the
// copies slow the short kernels more than the overlap gains.
static std::vector<uint64_t> stream_bounds(const hsdla_b200_engine* e, double rate, double fmul = 1.0,
                                           uint64_t min_first = 1) {
  const uint64_t na = e->na, nl = e->nl, ng = e->ng;
  std::vector<uint64_t> b{0};
  if (const char* plan = std::getenv("HSDLA_B200_STREAM_PLAN")) {  // explicit chunk sizes "4,9,19" (tuning)
    for (const char* c = plan; *c && b.back() < na;) {
      const uint64_t take = std::strtoull(c, const_cast<char**>(&c), 10);
      if (take == 0) break;
      b.push_back(std::min(na, b.back() + take));
      while (*c == ',') ++c;
    }
    if (b.back() < na) b.push_back(na);
    return b;
  }
  if (na * nl * ng < (uint64_t(1) << 22) || na < 2) {
    b.push_back(na);
    return b;
  }
  const double T = static_cast<double>(tiles_of(ng)), t0 = static_cast<double>(e->c0 / kTriBM),
               t1 = static_cast<double>(tiles_of(e->c1));
  const double tiles = (t1 - t0) * (t1 - t0 + 1) / 2 + (T - t1) * (t1 - t0);  // the window's lower tiles
  const double rows = static_cast<double>(e->row1 - e->row0) / static_cast<double>(na);  // contracted rows per atom
  // S and H: 2 segments of `rows` each over the window's tiles, 6 flops per complex MAC (3M)
  const double flops = 2.0 * 2.0 * 8.0 * rows * tiles * kTriBM * kTriBM * 0.75 +
                       32.0 * static_cast<double>(nl * nl * e->ncol) * 0.75;
  const double u = 2.0 * static_cast<double>(nl * e->ncol) * 16.0 / rate;
  const double c = flops / env_double("HSDLA_B200_STREAM_TFLOPS", 33e12);
  const double f = fmul * (50e-6 + static_cast<double>(e->npk) * 64.0 / 2e12);
  constexpr int kMaxChunks = 8;
  const size_t n = na;
  std::vector<double> best((kMaxChunks + 1) * (n + 1), 1e300);
  std::vector<uint32_t> from((kMaxChunks + 1) * (n + 1), 0);
  auto at = [&](int k, size_t m) { return static_cast<size_t>(k) * (n + 1) + m; };
  best[at(0, 0)] = 0.0;
  int kbest = 1;
  for (int k = 1; k <= kMaxChunks; ++k) {
    for (size_t m = 1; m <= n; ++m)
      for (size_t p = 0; p < m; ++p) {  // chunk k covers atoms [p, m)
        if (k == 1 && m < min_first && m < n) continue;
        const double prev = best[at(k - 1, p)];
        if (prev >= 1e299) continue;
        const double t = std::max(prev, u * static_cast<double>(m)) + c * static_cast<double>(m - p) + f;
        if (t < best[at(k, m)]) {
          best[at(k, m)] = t;
          from[at(k, m)] = static_cast<uint32_t>(p);
        }
      }
    if (best[at(k, n)] < best[at(kbest, n)]) kbest = k;
  }
  std::vector<uint64_t> cut(kbest + 1);
  cut[kbest] = n;
  for (int k = kbest; k > 0; --k) cut[k - 1] = from[at(k, cut[k])];
  if (trace_on()) {
    std::string pl;
    for (int k = 0; k < kbest; ++k) pl += std::to_string(cut[k + 1] - cut[k]) + (k + 1 < kbest ? "," : "");
    std::fprintf(stderr, "[hsdla_b200 trace] chunk plan at %.0f GB/s: %s (model %.2f ms)\n", rate / 1e9, pl.c_str(),
                 best[at(kbest, n)] * 1e3);
  }
  return cut;
}

// Tile-column boundaries splitting the window's lower tiles into kD2hPieces bands
// (column tj holds T - tj tiles); the packed range of band q is columns
// [64 c_q, 64 c_{q+1}).  Band q's download / reduce and host unpack run while band q+1
// computes, so only the last band's copy is exposed after the kernels end.  Band q+1
// holds kBandRatio x band q's tiles: 8 equal bands (ratio 1) measured best at C2
// (tools/stream_tune.py: 24.5 ms per call against 24.75 with 4 equal bands; shrinking
// bands, ratio 0.8 / 0.7, lost 0.1-0.6 ms because the small last launches run below
// full efficiency).
static void make_pieces(hsdla_b200_engine* e) {
  const double kBandRatio = env_double("HSDLA_B200_BAND_RATIO", 1.0);
  const long long T = static_cast<long long>(tiles_of(e->ng));
  const long long t0 = static_cast<long long>(e->c0 / kTriBM), t1 = static_cast<long long>(tiles_of(e->c1));
  long long total = 0;
  for (long long tj = t0; tj < t1; ++tj) total += T - tj;
  // 8 bands from 4 tile waves on; smaller triangles 3 (C1, 0.9 waves: 1.32 -> 1.20 ms per pinned call;
  // N_G 2000: 2.99 -> 2.86 ms; 2 and 4 bands measured in between)
  const int Qd = total >= 4LL * e->sms ? hsdla_b200_engine::kD2hPieces : 3;
  const int Q = std::max(1, std::min(hsdla_b200_engine::kD2hPieces, static_cast<int>(env_double("HSDLA_B200_BANDS", Qd))));
  double wsum = 0, w = 1;
  for (int q = 0; q < Q; ++q, w *= kBandRatio) wsum += w;
  e->piece_tiles[0] = static_cast<int>(t0);
  long long tj = t0, acc = 0;
  double cum = 0;
  w = 1;
  for (int q = 1; q < Q; ++q, w *= kBandRatio) {
    cum += w;
    const long long target = static_cast<long long>(static_cast<double>(total) * cum / wsum);
    while (tj < t1 && acc + (T - tj) <= target) acc += T - tj++;
    e->piece_tiles[q] = static_cast<int>(tj);
  }
  for (int q = Q; q <= hsdla_b200_engine::kD2hPieces; ++q) e->piece_tiles[q] = static_cast<int>(t1);
}

// The device-resident plans (set 0 and, when allocated, set 1); the streamed chunk
// plans are rebuilt lazily (ensure_streamed_plans) since a k-point batch reshaping the
// engine per k-point never uses them.
static void make_plans(hsdla_b200_engine* e) {
  make_pieces(e);
  e->whole.resize(1);
  make_chunk(e, 0, 0, e->na, true, e->whole[0]);
  if (e->Aset[1]) {
    e->whole2.resize(1);
    make_chunk(e, 1, 0, e->na, true, e->whole2[0]);
  }
  e->streamed_dirty = true;
}

void ensure_streamed_plans(hsdla_b200_engine* e) {
  if (!e->streamed_dirty) return;
  const auto b = stream_bounds(e, 50e9);
  e->streamed.resize(b.size() - 1);
  for (size_t c = 0; c + 1 < b.size(); ++c) make_chunk(e, 0, b[c], b[c + 1], c == 0, e->streamed[c]);
  // host-packed feeds (pageable rows packed into the slabs, HSDL files copied from the page
  // cache): ~35-44 GB/s, a chunk costs more (the host packs it before its launches are enqueued)
  // and the first one is at least N_A/16 (tools/small_probe.py, pageable: C2 20.7 ms per call
  // with 5,8,12,16,23 atoms against 20.9 for the earlier geometric 4,6,10,15,29; C3 180.0 against
  // 184.6 ms)
  const auto bp = stream_bounds(e, env_double("HSDLA_B200_PAGEABLE_RATE", 35e9), 2.0,
                                static_cast<uint64_t>(std::ceil(e->na / 16.0)));
  e->streamed_pg.resize(bp.size() - 1);
  for (size_t c = 0; c + 1 < bp.size(); ++c) make_chunk(e, 0, bp[c], bp[c + 1], c == 0, e->streamed_pg[c]);
  while (e->ev_chunk_up.size() < std::max(e->streamed.size(), e->streamed_pg.size())) {
    cudaEvent_t ev;
    HS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->ev_chunk_up.push_back(ev);
  }
  e->streamed_dirty = false;
}

// N_G = ng, window [c0, c1): fields and plans (capacity already checked).
static void set_geometry(hsdla_b200_engine* e, uint64_t ng, uint64_t c0, uint64_t c1) {
  e->ng = ng;
  e->c0 = c0;
  e->c1 = c1;
  e->ncol = ng - c0;
  e->pk0 = packed_col(ng, c0);
  e->npk = packed_col(ng, c1) - e->pk0;
  e->temp_bytes = e->K * e->ncol * sizeof(double2);
  make_plans(e);
}

// The second K x ncol temporary: Z next to T_AA A for the fused contraction, the
// Lft select for the original algorithm, W_B for the merged one.  Allocated once, then
// every plan is rebuilt against it.
static void ensure_x2(hsdla_b200_engine* e) {
  if (e->X2) return;
  HS_CUDA(cudaStreamSynchronize(e->stream));
  dalloc(e, &e->X2, e->K * e->cap_cols);
  make_plans(e);
}

hsdla_b200_engine* engine_create(int device, const ShardSpec& sp) {
  check_dims(sp.na, sp.nl, sp.ng);
  const uint64_t c1 = sp.c1 ? sp.c1 : sp.ng;
  check_window(sp.ng, sp.c0, c1);
  auto e = std::make_unique<hsdla_b200_engine>();
  e->device = device;
  e->na = sp.na;
  e->nl = sp.nl;
  e->K = sp.na * sp.nl;
  e->row0 = sp.row0;
  e->row1 = sp.row1 ? sp.row1 : e->K;
  if (e->row0 >= e->row1 || e->row1 > e->K || e->row0 >= sp.nl || e->row1 + sp.nl <= e->K)
    throw Fail{HSDLA_B200_CONFIG_ERROR, "row range [row0, row1) must lie in the shard and touch its first and last atom"};
  e->own_a0 = (e->row0 + sp.nl - 1) / sp.nl;
  e->own_a1 = (e->row1 + sp.nl - 1) / sp.nl;
  const bool all = sp.c0 == 0 && c1 == sp.ng;
  // capacity: a whole-window engine can be reshaped to any N_G up to ng_capacity
  const uint64_t cap_ng = all ? std::max(sp.ng, sp.ng_capacity) : sp.ng;
  check_dims(sp.na, sp.nl, cap_ng);
  e->cap_cols = cap_ng - sp.c0;
  e->cap_pk = all ? cap_ng * (cap_ng + 1) / 2 : packed_col(sp.ng, c1) - packed_col(sp.ng, sp.c0);
  try {
    HS_CUDA(cudaSetDevice(device));
    // Attributes are per-device for the current context: set them on every device.
    set_kernel_attributes();
    e->arith = g_default_arith.load();
    HS_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    HS_CUDA(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    HS_CUDA(cudaStreamCreateWithFlags(&e->comm_stream, cudaStreamNonBlocking));
    for (cudaEvent_t* ev : {&e->ev_begin, &e->ev_end_t, &e->ev_reduce_end, &e->ev_up0, &e->ev_up1, &e->ev_setup0,
                            &e->ev_setup1, &e->ev_setup_mid})
      HS_CUDA(cudaEventCreate(ev));
    for (cudaEvent_t* ev : {&e->ev_end, &e->ev_s_done, &e->ev_s_red, &e->ev_dl_s, &e->ev_a0, &e->ev_ops,
                            &e->ev_cs_order})
      HS_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    for (int q = 0; q < hsdla_b200_engine::kD2hPieces; ++q)
      for (cudaEvent_t* ev : {&e->ev_h_band[q], &e->ev_h_red[q], &e->ev_dl_h[q]})
        HS_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    for (auto& t : e->ring)
      for (cudaEvent_t* ev : {&t.s0, &t.s1, &t.h0, &t.h1}) HS_CUDA(cudaEventCreate(ev));
    const uint64_t KG = e->K * e->cap_cols, blk = sp.nl * sp.nl;
    dalloc(e.get(), &e->Aset[0], KG);
    dalloc(e.get(), &e->Bset[0], KG);
    dalloc(e.get(), &e->X1, KG);  // X2: on the first merged / fused / original build (ensure_x2)
    dalloc(e.get(), &e->Tab, sp.na * blk);
    dalloc(e.get(), &e->Taa, sp.na * blk);
    dalloc(e.get(), &e->Tbb, sp.na * blk);
    dalloc(e.get(), &e->Paa, sp.na * blk);
    dalloc(e.get(), &e->Pbb, sp.na * blk);
    dalloc(e.get(), &e->Wl, 4 * sp.na * blk);
    dalloc(e.get(), &e->U, e->K);
    dalloc(e.get(), &e->info, sp.na);
    dalloc(e.get(), &e->n_fail, 1);
    dalloc(e.get(), &e->Hp, e->cap_pk);
    dalloc(e.get(), &e->Sp, e->cap_pk);
    HS_CUDA(cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, device));
    dalloc(e.get(), &e->sk_ws, static_cast<uint64_t>(e->sms) * kSkSlot);
    dalloc(e.get(), &e->sk_flags, static_cast<uint64_t>(e->sms));
    HS_CUDA(cudaMemset(e->sk_flags, 0, e->sms * sizeof(uint32_t)));
    dalloc(e.get(), &e->d_stamp, static_cast<uint64_t>(hsdla_b200_engine::kMaxStamps) * kStampWords);
    HS_CUDA(cudaMemset(e->d_stamp, 0, hsdla_b200_engine::kMaxStamps * kStampWords * sizeof(unsigned long long)));
    set_geometry(e.get(), sp.ng, sp.c0, c1);
  } catch (...) {
    engine_free(e.get());
    throw;
  }
  return e.release();
}

bool engine_reshape(hsdla_b200_engine* e, uint64_t ng, uint64_t c0, uint64_t c1) {
  if (!c1) c1 = ng;
  check_dims(e->na, e->nl, ng);
  check_window(ng, c0, c1);
  if (ng == e->ng && c0 == e->c0 && c1 == e->c1) return true;
  if (ng - c0 > e->cap_cols || packed_col(ng, c1) - packed_col(ng, c0) > e->cap_pk) return false;
  HS_CUDA(cudaSetDevice(e->device));
  set_geometry(e, ng, c0, c1);
  return true;
}

static void check_problem(const hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0) {
  if (!p || !p->A || !p->B || !p->T_AA || !p->T_AB || !p->T_BB || !p->U)
    throw Fail{HSDLA_B200_DIMENSION_ERROR, "null problem pointer"};
  if (p->n_l != e->nl || p->n_g != e->ng || a0 + e->na > p->n_atoms)
    throw Fail{HSDLA_B200_DIMENSION_ERROR, "problem shape does not match the engine shard"};
}

// H2D of local atoms [b0, b1) (engine-local indices) of shard a0 of p into A/B set `set`,
// on stream s: the engine's columns [c0, p->n_g) of the caller's matrices.
// parts: 1 = A rows, 2 = B rows, 4 = operator blocks + U (7: everything)
static void upload_atoms(hsdla_b200_engine* e, int set, const hsdla_b200_problem* p, uint64_t a0, uint64_t b0,
                         uint64_t b1, cudaStream_t s, cudaEvent_t ev_a = nullptr, int parts = 7) {
  const uint64_t Kg = p->n_atoms * p->n_l;  // caller's leading dimension
  const uint64_t nl = e->nl, r0 = b0 * nl, rows = (b1 - b0) * nl, g0 = (a0 + b0) * nl;
  const uint64_t cols = p->n_g - e->c0, src0 = g0 + e->c0 * Kg;
  if (cols > e->cap_cols) throw Fail{HSDLA_B200_SIZING_ERROR, "problem exceeds the engine capacity"};
  const size_t width = rows * sizeof(double2);
  if (parts & 1)
    HS_CUDA(cudaMemcpy2DAsync(e->A(set) + r0, e->K * sizeof(double2), reinterpret_cast<const double2*>(p->A) + src0,
                              Kg * sizeof(double2), width, cols, cudaMemcpyHostToDevice, s));
  if (ev_a) HS_CUDA(cudaEventRecord(ev_a, s));
  if (parts & 2)
    HS_CUDA(cudaMemcpy2DAsync(e->B(set) + r0, e->K * sizeof(double2), reinterpret_cast<const double2*>(p->B) + src0,
                              Kg * sizeof(double2), width, cols, cudaMemcpyHostToDevice, s));
  if (!(parts & 4)) return;
  const uint64_t blk = nl * nl;
  const size_t tbytes = (b1 - b0) * blk * sizeof(double2);
  const uint64_t t0 = (a0 + b0) * blk;
  HS_CUDA(cudaMemcpyAsync(e->Taa + b0 * blk, reinterpret_cast<const double2*>(p->T_AA) + t0, tbytes,
                          cudaMemcpyHostToDevice, s));
  HS_CUDA(cudaMemcpyAsync(e->Tab + b0 * blk, reinterpret_cast<const double2*>(p->T_AB) + t0, tbytes,
                          cudaMemcpyHostToDevice, s));
  HS_CUDA(cudaMemcpyAsync(e->Tbb + b0 * blk, reinterpret_cast<const double2*>(p->T_BB) + t0, tbytes,
                          cudaMemcpyHostToDevice, s));
  HS_CUDA(cudaMemcpyAsync(e->U + r0, p->U + g0, rows * sizeof(double), cudaMemcpyHostToDevice, s));
}

void engine_fill_synthetic(hsdla_b200_engine* e, uint64_t seed) {
  HS_CUDA(cudaSetDevice(e->device));
  const unsigned grid = static_cast<unsigned>(e->sms * 8);
  auto fill = [&](void* ptr, uint64_t n, uint64_t salt, double lo, double hi) {
    launch_fill_uniform(static_cast<double*>(ptr), n, seed * 16 + salt, lo, hi, grid, e->stream);
  };
  const uint64_t KG2 = 2 * e->K * e->ncol, T2 = 2 * e->na * e->nl * e->nl;
  fill(e->A(0), KG2, 1, -1.0, 1.0);
  fill(e->B(0), KG2, 2, -1.0, 1.0);
  fill(e->Taa, T2, 3, -1.0, 1.0);
  fill(e->Tab, T2, 4, -1.0, 1.0);
  fill(e->Tbb, T2, 5, -1.0, 1.0);
  fill(e->U, e->K, 6, 0.5, 1.5);
}

// Staging ring of pinned slabs owned by the engine; slab s is free again once the copy
// that read it has completed.
char* stage_acquire(hsdla_b200_engine* e, int& slot) {
  if (!e->stage_buf[0])
    for (int i = 0; i < hsdla_b200_engine::kStageSlabs; ++i) {
      HS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&e->stage_buf[i]), kStageSlab));
      HS_CUDA(cudaEventCreateWithFlags(&e->stage_ev[i], cudaEventDisableTiming));
    }
  slot = e->stage_next;
  e->stage_next = (e->stage_next + 1) % hsdla_b200_engine::kStageSlabs;
  if (e->stage_busy[slot]) {
    const double t0 = trace_on() ? host_ms() : 0.0;
    HS_CUDA(cudaEventSynchronize(e->stage_ev[slot]));
    if (trace_on()) e->tr_wait_ms += host_ms() - t0;
  }
  e->stage_busy[slot] = true;
  return e->stage_buf[slot];
}
void stage_release(hsdla_b200_engine* e, int slot, cudaStream_t s) {
  HS_CUDA(cudaEventRecord(e->stage_ev[slot], s));
}

// True if [p, p + bytes) is page-locked host memory (registered or cudaMallocHost).
static bool is_pinned(const void* p, size_t bytes) {
  if (!p || !bytes) return true;
  cudaPointerAttributes a0{}, a1{};
  const void* last = static_cast<const char*>(p) + bytes - 1;
  if (cudaPointerGetAttributes(&a0, p) != cudaSuccess || cudaPointerGetAttributes(&a1, last) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a0.type == cudaMemoryTypeHost && a1.type == cudaMemoryTypeHost;
}

static void stage_operator_blocks(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0, uint64_t b0,
                                  uint64_t b1, cudaStream_t s);
static void stage_u(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0, uint64_t b0, uint64_t b1,
                    cudaStream_t s);

// upload_atoms for PAGEABLE caller buffers: the rows of atoms [b0, b1) are packed by up
// to 16 host threads into the engine's pinned staging slabs and copied from there
// (a pageable cudaMemcpy is host-synchronous and single-threaded, ~10 GB/s).
// parts: 1 = A rows, 2 = B rows, 4 = operator blocks + U (7: everything)
static void upload_atoms_staged(hsdla_b200_engine* e, int set, const hsdla_b200_problem* p, uint64_t a0,
                                uint64_t b0, uint64_t b1, cudaStream_t s, int parts = 7) {
  const uint64_t Kg = p->n_atoms * p->n_l, nl = e->nl;
  const uint64_t r0 = b0 * nl, rows = (b1 - b0) * nl, g0 = (a0 + b0) * nl;
  const uint64_t cols = p->n_g - e->c0, src0 = g0 + e->c0 * Kg;
  if (cols > e->cap_cols) throw Fail{HSDLA_B200_SIZING_ERROR, "problem exceeds the engine capacity"};
  const size_t colb = rows * sizeof(double2);
  for (int m = 0; m < 2; ++m) {
    if (!(parts & (m == 0 ? 1 : 2))) continue;
    const double2* src = reinterpret_cast<const double2*>(m == 0 ? p->A : p->B) + src0;
    double2* dst = (m == 0 ? e->A(set) : e->B(set)) + r0;
    if (colb > kStageSlab) {  // one column's rows exceed a slab: direct (pageable) copy
      HS_CUDA(cudaMemcpy2DAsync(dst, e->K * sizeof(double2), src, Kg * sizeof(double2), colb, cols,
                                cudaMemcpyHostToDevice, s));
      continue;
    }
    // pack pieces of ~1/div of the matrix (1 MB .. one slab): the DMA of piece i overlaps
    // the packing of piece i+1
    static const double div = std::max(1.0, env_double("HSDLA_B200_PIECE_DIV", 4.0));
    const size_t sp = slab_pitch(colb);  // each column's rows on a 4 KB boundary of the slab
    const uint64_t piece = std::min<uint64_t>(kStageSlab, std::max<uint64_t>(uint64_t(1) << 20,
                                              static_cast<uint64_t>(static_cast<double>(sp * cols) / div)));
    const uint64_t per = std::max<uint64_t>(1, piece / sp);
    for (uint64_t j0 = 0; j0 < cols; j0 += per) {
      const uint64_t nc = std::min(per, cols - j0);
      int slot;
      char* b = stage_acquire(e, slot);
      const double t0 = trace_on() ? host_ms() : 0.0;
      par_for(nc, nc * colb, [&](uint64_t j) { copy_nt(b + j * sp, src + (j0 + j) * Kg, colb); });
      _mm_sfence();  // the single-threaded case of par_for
      if (trace_on()) {
        e->tr_pack_ms += host_ms() - t0;
        e->tr_pack_bytes += nc * colb;
      }
      HS_CUDA(cudaMemcpy2DAsync(dst + j0 * e->K, e->K * sizeof(double2), b, sp, colb, nc, cudaMemcpyHostToDevice,
                                s));
      stage_release(e, slot, s);
    }
  }
  if (!(parts & 4)) return;
  stage_operator_blocks(e, p, a0, b0, b1, s);
  stage_u(e, p, a0, b0, b1, s);
}

// The operator blocks (T_AA, T_AB, T_BB) of local atoms [b0, b1) through the slabs: groups of
// atoms whose three blocks fit one slab (large chunks of large-N_L atoms need several).
static void stage_operator_blocks(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0, uint64_t b0,
                                  uint64_t b1, cudaStream_t s) {
  const uint64_t nl = e->nl, blk = nl * nl, bb = blk * sizeof(double2);
  if (3 * bb > kStageSlab) throw Fail{HSDLA_B200_SIZING_ERROR, "operator blocks larger than the staging slab"};
  const uint64_t per = std::max<uint64_t>(1, kStageSlab / (3 * bb));
  const double* srcs[3] = {p->T_AA, p->T_AB, p->T_BB};
  double2* dsts[3] = {e->Taa, e->Tab, e->Tbb};
  for (uint64_t c0 = b0; c0 < b1; c0 += per) {
    const uint64_t nb = std::min(per, b1 - c0);
    const size_t tb = nb * bb;
    int slot;
    char* b = stage_acquire(e, slot);
    par_for(3, 3 * tb, [&](uint64_t m) {
      copy_nt(b + m * tb, reinterpret_cast<const double2*>(srcs[m]) + (a0 + c0) * blk, tb);
    });
    _mm_sfence();
    for (int m = 0; m < 3; ++m)
      HS_CUDA(cudaMemcpyAsync(dsts[m] + c0 * blk, b + m * tb, tb, cudaMemcpyHostToDevice, s));
    stage_release(e, slot, s);
  }
}

// U of local atoms [b0, b1) through a slab.
static void stage_u(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0, uint64_t b0, uint64_t b1,
                    cudaStream_t s) {
  const uint64_t nl = e->nl, r0 = b0 * nl, rows = (b1 - b0) * nl, g0 = (a0 + b0) * nl;
  const size_t ub = rows * sizeof(double);
  if (ub > kStageSlab) throw Fail{HSDLA_B200_SIZING_ERROR, "U larger than the staging slab"};
  int slot;
  char* b = stage_acquire(e, slot);
  std::memcpy(b, p->U + g0, ub);
  HS_CUDA(cudaMemcpyAsync(e->U + r0, b, ub, cudaMemcpyHostToDevice, s));
  stage_release(e, slot, s);
}

void engine_upload(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0) {
  check_problem(e, p, a0);
  HS_CUDA(cudaSetDevice(e->device));
  upload_atoms(e, 0, p, a0, 0, e->na, e->stream);
}

// ---- launches ---------------------------------------------------------------
// The next `n` launch timestamp slots (stamp.cuh), or nullptr (untimed launch) once the build
// has used them all; take_stamp commits one slot, launches that may use up to n commit what they used.
static unsigned long long* stamp_slots(hsdla_b200_engine* e, int n) {
  return e->stamp_used + n <= hsdla_b200_engine::kMaxStamps ? e->d_stamp + e->stamp_used * kStampWords : nullptr;
}
static unsigned long long* take_stamp(hsdla_b200_engine* e) {
  unsigned long long* p = stamp_slots(e, 1);
  if (p) ++e->stamp_used;
  return p;
}
// A launcher that may launch nothing (an empty range) takes a slot only when it launched, so no
// slot keeps an earlier build's times.
template <class F>
static void stamped(hsdla_b200_engine* e, F&& launch) {
  unsigned long long* p = stamp_slots(e, 1);
  if (launch(p) && p) ++e->stamp_used;
}

// Build brackets.  ev_end orders the downloads after the build; the timing events exist for the
// reduce's timeline only (a timing event on the compute stream costs 30-55 us while a copy is in
// flight, stamp.cuh), so engines that never reduce with others skip them.
static bool grouped(const hsdla_b200_engine* e) { return e->comm || !e->local_group.empty(); }
void mark_build_begin(hsdla_b200_engine* e) {
  e->marks_timed = grouped(e);
  if (e->marks_timed) HS_CUDA(cudaEventRecord(e->ev_begin, e->stream));
}
void mark_build_end(hsdla_b200_engine* e) {
  HS_CUDA(cudaEventRecord(e->ev_end, e->stream));
  if (e->marks_timed) HS_CUDA(cudaEventRecord(e->ev_end_t, e->stream));
}

void copy_after_compute(hsdla_b200_engine* e) {
  HS_CUDA(cudaEventRecord(e->ev_cs_order, e->stream));
  HS_CUDA(cudaStreamWaitEvent(e->copy_stream, e->ev_cs_order, 0));
}

// HSDLA_B200_TRACE: a timing event on stream s named `what` (device timeline of one call).
void trace_mark(hsdla_b200_engine* e, cudaStream_t s, const std::string& what) {
  if (!trace_on()) return;
  if (e->tr_marks.size() == e->tr_pool.size()) {
    cudaEvent_t ev;
    HS_CUDA(cudaEventCreate(&ev));
    e->tr_pool.push_back(ev);
  }
  cudaEvent_t ev = e->tr_pool[e->tr_marks.size()];
  HS_CUDA(cudaEventRecord(ev, s));
  e->tr_marks.push_back({what, ev});
}

// NVTX range names of the phase slots (include/hsdla_b200.h HSDLA_B200_PHASE_*).
static const char* const kPhaseNames[HSDLA_B200_N_PHASES] = {"s",         "z_loop",    "her2k",       "hemm_loop",
                                                             "herkx",     "chol_loop", "h_aa_update", "-"};

// One phase op on the compute stream: the launch timestamp slots its kernels take (plus an NVTX
// range around its enqueue, for nsys / ncu --nvtx timelines).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
template <class F>
static void timed_op(hsdla_b200_engine* e, int phase, F&& body) {
  NvtxRange range(kPhaseNames[phase]);
  const int s0 = e->stamp_used;
  body();
  e->ops.push_back({phase, s0, e->stamp_used});
}

static void launch_tri(hsdla_b200_engine* e, const CtnParams& P, const dim3& grid) {
  CtnParams q = P;
  q.epoch = ++e->epoch;  // fresh stream-K flag generation per launch
  q.stamp = stamp_slots(e, 3);  // up to 3 kernels (strictly-lower, ragged row, diagonal)
  const int n = launch_tri_kernel(e->arith, grid, q, e->stream);
  e->launches += n;
  if (q.stamp) e->stamp_used += n;
}
static void launch_bat(hsdla_b200_engine* e, const CtnParams& P, const dim3& grid) {
  CtnParams q = P;
  q.stamp = take_stamp(e);
  launch_bat_kernel(e->arith, grid, q, e->stream);
  ++e->launches;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  HS_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

void harvest(hsdla_b200_engine* e, hsdla_b200_engine::KTimer& t) {
  if (!t.pending) return;
  HS_CUDA(cudaEventSynchronize(t.h1));
  e->sum_s_ms += ev_ms(t.s0, t.s1);
  e->sum_h_ms += ev_ms(t.h0, t.h1);
  e->sum_flops_h += t.flops_h;
  e->sum_flops_s += t.flops_s;
  ++e->timed_builds;
  t.pending = false;
}

// All phases of one chunk on the compute stream, in the reference phase order of
// the chosen algorithm:
//   refined  s, z_loop, her2k, hemm_loop, herkx        (pipeline.cpp:281-329), one temp X1
//   fused    s, z_loop, hemm_loop, her2k(+herkx)       two temps (Z in X2)
//   merged   s, z_loop (W_A, W_B), her2k (one H contraction)
//   original z_loop, her2k, s, chol_loop, h_aa_update  (pipeline.cpp:189-279), two temps
// s_rest: the chunk's A^H A half of S already ran (enqueue_s_first); phase s adds (UB)^H (UB).
void enqueue_chunk(hsdla_b200_engine* e, ChunkPlan& cp, int algo, bool last, hsdla_b200_engine::KTimer* kt,
                   bool s_rest) {
  cudaStream_t s = e->stream;
  // The build's final H contraction: whole, or band by band (tile-column bands of
  // equal work, event after each; make_pieces) so the download / reduce of band q
  // overlaps band q+1.
  auto final_h = [&](const CtnParams& P) {
    if (e->wait_before_h) HS_CUDA(cudaStreamWaitEvent(s, e->wait_before_h, 0));  // H storage reuse
    // bands: the one-shot drop-in (download overlaps) and every multi-rank build (the
    // reduce of band q overlaps the compute of band q+1)
    // (from half a tile wave on; below 4 waves in 3 bands, make_pieces)
    static const double min_waves = env_double("HSDLA_B200_BAND_MIN_WAVES", 0.5);
    if (!(last && (e->band_final_h || grouped(e)) && P.tiles_total >= min_waves * e->sms)) {
      launch_tri(e, P, cp.grid_tri);
      return;
    }
    int iters = 0;
    for (int sg = 0; sg < P.nseg; ++sg) iters += P.kchunks[sg];
    const int T = P.tiles;
    for (int q = 0; q < hsdla_b200_engine::kD2hPieces; ++q) {
      const int c0 = e->piece_tiles[q], c1 = e->piece_tiles[q + 1];
      long long cnt = 0;
      for (int tj = c0; tj < c1; ++tj) cnt += T - tj;
      if (cnt > 0) {
        CtnParams b = P;
        b.col_t0 = c0;
        b.col_t1 = c1;
        b.tiles_total = static_cast<int>(cnt);
        const dim3 g(static_cast<unsigned>(std::min<long long>(e->sms, cnt * iters)));
        launch_tri(e, b, g);
      }
      HS_CUDA(cudaEventRecord(e->ev_h_band[q], s));
    }
    e->banded = true;
  };
  const uint64_t nac = cp.a1 - cp.a0, nl = e->nl, r0 = cp.a0 * nl, Kc = nac * nl, ncol = e->ncol;
  auto expand = [&] {
    // operator expansion (lower triangles of T_AA, T_BB only) for this chunk's atoms
    const uint64_t total = nac * nl * nl, off = cp.a0 * nl * nl;
    const bool merged = algo == HSDLA_B200_ALGO_REFINED_MERGED;
    stamped(e, [&](unsigned long long* st) {
      return launch_expand_hermitian(e->Taa + off, e->Tbb + off, e->Paa + off, e->Pbb + off, static_cast<int>(nl),
                                     total, merged ? 1.0 : 0.5, e->Tab + off, merged ? e->Wl + 4 * off : nullptr, s,
                                     st);
    });
    ++e->launches;
  };
  // operators uploaded on the copy stream (engine_upload_operators): wait before expanding
  auto expand_ops = [&] {
    if (e->ops_pending) HS_CUDA(cudaStreamWaitEvent(s, e->ev_ops, 0));
    expand();
  };
  auto phase_s = [&] {
    timed_op(e, HSDLA_B200_PHASE_S, [&] {
      if (e->wait_before_s) HS_CUDA(cudaStreamWaitEvent(s, e->wait_before_s, 0));
      stamped(e, [&](unsigned long long* st) {
        return launch_diag_scale(cp.B + r0, e->U + r0, e->X1 + r0, Kc, e->K, ncol, s, st);
      });
      ++e->launches;
      if (kt) HS_CUDA(cudaEventRecord(kt->s0, s));
      launch_tri(e, s_rest ? cp.sB : cp.s, cp.grid_tri);
      if (kt) HS_CUDA(cudaEventRecord(kt->s1, s));
    });
    if (last) HS_CUDA(cudaEventRecord(e->ev_s_done, s));
    if (last) trace_mark(e, s, "s_done");
  };
  auto timed_h = [&](CtnParams& P, bool final) {
    if (e->wait_before_h) HS_CUDA(cudaStreamWaitEvent(s, e->wait_before_h, 0));  // H storage reuse
    if (kt) HS_CUDA(cudaEventRecord(kt->h0, s));
    if (final)
      final_h(P);
    else
      launch_tri(e, P, cp.grid_tri);
    if (kt) HS_CUDA(cudaEventRecord(kt->h1, s));
  };
  if (algo == HSDLA_B200_ALGO_ORIGINAL) {
    timed_op(e, HSDLA_B200_PHASE_Z_LOOP, [&] {
      expand_ops();
      launch_bat(e, cp.z, cp.grid_bat);
    });
    timed_op(e, HSDLA_B200_PHASE_HER2K, [&] { timed_h(cp.h2k, false); });
    phase_s();
    timed_op(e, HSDLA_B200_PHASE_CHOL_LOOP, [&] {
      if (cp.a0 == 0) HS_CUDA(cudaMemsetAsync(e->n_fail, 0, sizeof(int), s));  // first chunk of the build
      stamped(e, [&](unsigned long long* st) {
        return launch_potrf_batched(e->Taa + cp.a0 * nl * nl, e->Paa + cp.a0 * nl * nl, e->info + cp.a0,
                                    static_cast<int>(nl), nac, e->n_fail, s, st);
      });
      ++e->launches;
      launch_bat(e, cp.x, cp.grid_bat);  // W_a = Q_a^H A_a: trmm (HPD) or hemm (failed)
      stamped(e, [&](unsigned long long* st) {
        return launch_select_left(e->X1 + r0, cp.A + r0, e->info + cp.a0, e->X2 + r0, Kc, e->K, ncol,
                                  static_cast<int>(nl), s, st);
      });
      ++e->launches;
    });
    timed_op(e, HSDLA_B200_PHASE_H_AA_UPDATE, [&] { final_h(cp.haa); });
    return;
  }
  // S needs no operator: it runs before the expansion (and, after an operator upload on the
  // copy stream, while the operators travel)
  phase_s();
  if (algo == HSDLA_B200_ALGO_REFINED) {
    timed_op(e, HSDLA_B200_PHASE_Z_LOOP, [&] {
      expand_ops();
      launch_bat(e, cp.z, cp.grid_bat);
    });
    timed_op(e, HSDLA_B200_PHASE_HER2K, [&] { timed_h(cp.h2k, false); });
    timed_op(e, HSDLA_B200_PHASE_HEMM_LOOP, [&] { launch_bat(e, cp.x, cp.grid_bat); });
    timed_op(e, HSDLA_B200_PHASE_HERKX, [&] { final_h(cp.hkx); });
  } else if (algo == HSDLA_B200_ALGO_REFINED_MERGED) {
    timed_op(e, HSDLA_B200_PHASE_Z_LOOP, [&] {
      expand_ops();
      trace_mark(e, s, "x");
      CtnParams w = cp.w;
      w.stamp = take_stamp(e);
      launch_batw_kernel(e->arith, cp.w_bn, cp.grid_batw, w, e->stream);  // W_A and W_B
      ++e->launches;
      trace_mark(e, s, "w");
    });
    timed_op(e, HSDLA_B200_PHASE_HER2K, [&] { timed_h(cp.hm, true); });  // her2k + herkx merged
  } else {
    timed_op(e, HSDLA_B200_PHASE_Z_LOOP, [&] {
      expand_ops();
      launch_bat(e, cp.zf, cp.grid_bat);
    });
    timed_op(e, HSDLA_B200_PHASE_HEMM_LOOP, [&] { launch_bat(e, cp.x, cp.grid_bat); });
    timed_op(e, HSDLA_B200_PHASE_HER2K, [&] { timed_h(cp.h, true); });  // her2k + herkx fused
  }
}

// The first streamed chunk's A^H A half of S, enqueued as soon as its A rows landed (the
// stream already waits for them): it overlaps the upload of B, T and U.
static void enqueue_s_first(hsdla_b200_engine* e, ChunkPlan& cp) {
  timed_op(e, HSDLA_B200_PHASE_S, [&] { launch_tri(e, cp.sA, cp.grid_tri); });
}

void begin_build(hsdla_b200_engine* e, int algo) {
  if (!valid_algo(algo)) throw Fail{HSDLA_B200_CONFIG_ERROR, "unknown algo " + std::to_string(algo)};
  HS_CUDA(cudaSetDevice(e->device));
  if (algo != HSDLA_B200_ALGO_REFINED) ensure_x2(e);
  e->launches = 0;
  e->last_algo = algo;
  e->reduced = false;
  e->uploaded_streamed = false;
  e->stamp_used = 0;
  e->marks_timed = false;
  e->ops.clear();
  e->tr_marks.clear();
  e->built = true;
  e->banded = false;
  if (e->overlap_dl) e->band_final_h = true;  // (the one-shot drop-in sets and clears it itself)
}

// Device-resident build: one chunk over all atoms (the bench's `value`).
void engine_build(hsdla_b200_engine* e, int algo) {
  begin_build(e, algo);
  auto& kt = e->ring[e->builds++ % hsdla_b200_engine::kRing];
  harvest(e, kt);
  const uint64_t rows = e->row1 - e->row0;
  kt.flops_h = (algo == HSDLA_B200_ALGO_REFINED_FUSED ? 12 : 8) * rows * e->ng * e->ng;
  kt.flops_s = 8 * rows * e->ng * e->ng;
  if (!whole(e)) {  // a window's share of the triangle (executed tiles; ledger-style count)
    const double f = static_cast<double>(e->npk) / (static_cast<double>(e->ng) * (e->ng + 1) / 2);
    kt.flops_h = static_cast<uint64_t>(kt.flops_h * f);
    kt.flops_s = static_cast<uint64_t>(kt.flops_s * f);
  }
  mark_build_begin(e);
  // HSDLA_B200_CHUNKED_BUILD=1 (tuning): the device-resident inputs in the streamed drop-in's
  // atom chunks (the chunking's own cost, without the uploads)
  static const bool chunked = env_double("HSDLA_B200_CHUNKED_BUILD", 0) != 0;
  if (chunked && whole(e)) {
    ensure_streamed_plans(e);
    for (size_t c = 0; c < e->streamed.size(); ++c)
      enqueue_chunk(e, e->streamed[c], algo, c + 1 == e->streamed.size(), c + 1 == e->streamed.size() ? &kt : nullptr);
  } else {
    enqueue_chunk(e, e->whole[0], algo, true, &kt);
  }
  e->ops_pending = false;
  mark_build_end(e);
  kt.pending = true;
}

// Streamed build from host memory: chunk c+1's H2D overlaps chunk c's phases.
void engine_build_streamed(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0, int algo) {
  check_problem(e, p, a0);
  begin_build(e, algo);
  ensure_streamed_plans(e);
  // the copy stream may only overwrite A/B/T/U once the previous build has consumed them (and
  // after any upload still in flight on the compute stream)
  copy_after_compute(e);
  HS_CUDA(cudaEventRecord(e->ev_up0, e->copy_stream));
  trace_mark(e, e->copy_stream, "up_start");
  const uint64_t ab_bytes = p->n_atoms * p->n_l * p->n_g * sizeof(double2);
  const bool pinned = is_pinned(p->A, ab_bytes) && is_pinned(p->B, ab_bytes);
  // pageable rows are packed into pinned slabs by the host pool and DMA'd from there: the
  // host-packed plan (HSDLA_B200_PAGEABLE_PLAN=pinned: the page-locked one)
  const char* pgp = std::getenv("HSDLA_B200_PAGEABLE_PLAN");
  auto& plan = pinned || (pgp && std::strcmp(pgp, "pinned") == 0) ? e->streamed : e->streamed_pg;
  // The first chunk's S starts with its A^H A half as soon as A's rows landed, hiding part
  // of the one upload nothing can overlap (not for the original algorithm, whose first
  // phase needs B and T; HSDLA_B200_SPLIT_S=0 disables it for comparisons)
  const char* sp = std::getenv("HSDLA_B200_SPLIT_S");
  const bool split = algo != HSDLA_B200_ALGO_ORIGINAL && !(sp && *sp == '0');
  if (pinned) {
    // page-locked inputs: every chunk's copies are asynchronous, enqueue them all first.  The
    // small operator blocks and U of a caller who registered only A and B go through the
    // staging slabs: a pageable cudaMemcpyAsync would block the host until the copy stream
    // drained, serialising every upload before the first launch.
    const uint64_t blk_bytes = p->n_atoms * p->n_l * p->n_l * sizeof(double2);
    const bool ops_pinned = is_pinned(p->T_AA, blk_bytes) && is_pinned(p->T_AB, blk_bytes) &&
                            is_pinned(p->T_BB, blk_bytes) && is_pinned(p->U, p->n_atoms * p->n_l * sizeof(double));
    // Unregistered operators: every atom's U goes up with chunk 0's rows (phase s needs it) and
    // every atom's operator blocks right after them, staged ONCE through as few slabs as hold
    // them; the expansions wait on ev_ops.  (Staged chunk by chunk, a later chunk's slab waited
    // for a DMA queued behind the earlier chunks' A, B rows, blocking this host loop — and the
    // first launch — for milliseconds: C2 22.0 ms per call.)
    for (size_t c = 0; c < plan.size(); ++c) {
      upload_atoms(e, 0, p, a0, plan[c].a0, plan[c].a1, e->copy_stream, c == 0 && split ? e->ev_a0 : nullptr,
                   ops_pinned ? 7 : 3);
      if (c == 0 && !ops_pinned) stage_u(e, p, a0, 0, e->na, e->copy_stream);
      HS_CUDA(cudaEventRecord(e->ev_chunk_up[c], e->copy_stream));
      if (trace_on()) trace_mark(e, e->copy_stream, "up" + std::to_string(c));
      if (c == 0 && !ops_pinned) {
        stage_operator_blocks(e, p, a0, 0, e->na, e->copy_stream);
        HS_CUDA(cudaEventRecord(e->ev_ops, e->copy_stream));
        e->ops_pending = true;
      }
    }
  }
  for (size_t c = 0; c < plan.size(); ++c) {
    const bool first_split = c == 0 && split;
    if (first_split) {
      if (!pinned) {
        upload_atoms_staged(e, 0, p, a0, plan[c].a0, plan[c].a1, e->copy_stream, 1);
        HS_CUDA(cudaEventRecord(e->ev_a0, e->copy_stream));
      }
      HS_CUDA(cudaStreamWaitEvent(e->stream, e->ev_a0, 0));
      mark_build_begin(e);
      enqueue_s_first(e, plan[c]);
    }
    if (!pinned) {
      // pageable inputs: the host packs chunk c into the pinned slabs while the GPU
      // already computes chunk c-1 (its phases were enqueued in the previous iteration)
      upload_atoms_staged(e, 0, p, a0, plan[c].a0, plan[c].a1, e->copy_stream, first_split ? 6 : 7);
      HS_CUDA(cudaEventRecord(e->ev_chunk_up[c], e->copy_stream));
      if (trace_on()) trace_mark(e, e->copy_stream, "up" + std::to_string(c));
    }
    HS_CUDA(cudaStreamWaitEvent(e->stream, e->ev_chunk_up[c], 0));
    if (c == 0 && !first_split) mark_build_begin(e);
    if (trace_on()) trace_mark(e, e->stream, "c" + std::to_string(c) + "_start");
    enqueue_chunk(e, plan[c], algo, c + 1 == plan.size(), nullptr, first_split);
    if (trace_on()) trace_mark(e, e->stream, "c" + std::to_string(c) + "_end");
  }
  HS_CUDA(cudaEventRecord(e->ev_up1, e->copy_stream));
  mark_build_end(e);
  e->ops_pending = false;  // every expansion of this build waited for them
  e->uploaded_streamed = true;
  if (trace_on() && !pinned) {
    std::fprintf(stderr, "[hsdla_b200 trace] pageable staging: packed %.0f MB in %.1f ms (%.1f GB/s), waited %.1f ms "
                 "for slabs, %zu chunks\n", e->tr_pack_bytes / 1e6, e->tr_pack_ms,
                 e->tr_pack_bytes / std::max(e->tr_pack_ms, 1e-9) / 1e6, e->tr_wait_ms, plan.size());
    e->tr_pack_ms = e->tr_wait_ms = 0;
    e->tr_pack_bytes = 0;
  }
}

// ---- k-point batches -----------------------------------------------------------------
// A/B set 1, the upload stream and its events, allocated all-or-nothing (a failure leaves
// the engine exactly as it was, set 1 absent).
static void ensure_kpoints(hsdla_b200_engine* e, int algo) {
  if (algo != HSDLA_B200_ALGO_REFINED) ensure_x2(e);
  if (e->Aset[1]) return;
  HS_CUDA(cudaStreamSynchronize(e->stream));
  double2 *a = nullptr, *b = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[4] = {};
  const size_t bytes = e->K * e->cap_cols * sizeof(double2);
  auto undo = [&] {
    if (a) cudaFree(a);
    if (b) cudaFree(b);
    if (st) cudaStreamDestroy(st);
    for (cudaEvent_t x : ev)
      if (x) cudaEventDestroy(x);
  };
  try {
    HS_CUDA(cudaMalloc(reinterpret_cast<void**>(&a), std::max<size_t>(bytes, 16)));
    HS_CUDA(cudaMalloc(reinterpret_cast<void**>(&b), std::max<size_t>(bytes, 16)));
    HS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (cudaEvent_t& x : ev) HS_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  } catch (...) {
    undo();
    throw;
  }
  e->Aset[1] = a;
  e->Bset[1] = b;
  e->device_bytes += 2 * std::max<size_t>(bytes, 16);
  e->h2d_stream = st;
  e->ev_kup[0] = ev[0];
  e->ev_kup[1] = ev[1];
  e->ev_kbuilt[0] = ev[2];
  e->ev_kbuilt[1] = ev[3];
  make_plans(e);
}

// n_k k-points of one cell: the operators and U are k-independent (uploaded once), A_k and
// B_k (N_G(k) = ngk[k] columns; ngk null: the cell's n_g) alternate between the two device
// sets.  While k-point k builds, the next one's A, B go up on the upload stream (or are packed
// into the staging slabs by the host) and k-1's H, S come down and are unpacked; the
// per-k-point cost approaches the device-resident build.  The engine's capacity must hold
// the largest N_G(k) (the caller sizes it).
void engine_kpoints(hsdla_b200_engine* e, const hsdla_b200_problem* common, uint64_t nk, const uint64_t* ngk,
                    const double* const* A, const double* const* B, int algo, double* const* H, double* const* S) {
  if (!whole(e)) throw Fail{HSDLA_B200_CONFIG_ERROR, "k-point batches need a whole-window engine"};
  auto ng_of = [&](uint64_t k) { return ngk ? ngk[k] : common->n_g; };
  for (uint64_t k = 0; k < nk; ++k)
    if (ng_of(k) < 1 || ng_of(k) > e->cap_cols) throw Fail{HSDLA_B200_SIZING_ERROR, "N_G(k) exceeds the engine capacity"};
  ensure_kpoints(e, algo);
  // download slots in rotation: k-point k downloads into slot k % depth and the host unpacks
  // k - depth + 1 after enqueueing build k and k's D2H.  Depth 3 keeps the next build queued
  // on the GPU while the host unpacks (small cells: the host loop, not the GPU, set the pace
  // at depth 2); large stages (> 256 MB pinned each) stay at 2, their builds hide the unpack.
  const double slot_mb = env_double("HSDLA_B200_KPOINT_SLOT_MB", 256.0);
  const int depth = 2 * e->cap_pk * sizeof(double2) <= slot_mb * (1 << 20) ? hsdla_b200_engine::kDlSlots : 2;
  auto slot_of = [&](uint64_t k) { return static_cast<int>(k % depth); };
  auto upload = [&](uint64_t k) {
    hsdla_b200_problem pk = *common;
    pk.A = A[k];
    pk.B = B[k];
    pk.n_g = ng_of(k);
    const size_t ab_bytes = e->K * pk.n_g * sizeof(double2);
    const int set = static_cast<int>(k & 1);
    HS_CUDA(cudaStreamWaitEvent(e->h2d_stream, e->ev_kbuilt[set], 0));  // k-2 is done with this set
    if (is_pinned(A[k], ab_bytes) && is_pinned(B[k], ab_bytes))
      upload_atoms(e, set, &pk, 0, 0, e->na, e->h2d_stream, nullptr, 3);
    else
      upload_atoms_staged(e, set, &pk, 0, 0, e->na, e->h2d_stream, 3);
    HS_CUDA(cudaEventRecord(e->ev_kup[set], e->h2d_stream));
  };
  for (uint64_t k = 0; k < nk; ++k) {
    const int set = static_cast<int>(k & 1);
    if (!engine_reshape(e, ng_of(k))) throw Fail{HSDLA_B200_SIZING_ERROR, "N_G(k) exceeds the engine capacity"};
    if (k == 0) {
      // the first k-point streams in atom chunks like the per-call drop-in (its upload
      // overlaps its own build); it also brings T and U, which every later k-point reuses
      hsdla_b200_problem p0 = *common;
      p0.A = A[0];
      p0.B = B[0];
      p0.n_g = ng_of(0);
      e->band_final_h = nk == 1 || env_double("HSDLA_B200_KPOINT_BANDS", 0) != 0;
      try {
        engine_build_streamed(e, &p0, 0, algo);
      } catch (...) {
        e->band_final_h = false;
        throw;
      }
      e->band_final_h = false;
      HS_CUDA(cudaEventRecord(e->ev_kbuilt[0], e->stream));
      if (nk > 1) upload(1);
      enqueue_download(e);
      continue;
    }
    begin_build(e, algo);
    // only the last k-point's final H runs in bands: every earlier download overlaps the next
    // build anyway, and the bands' launches cost ~1 % of a build
    e->band_final_h = k + 1 == nk || env_double("HSDLA_B200_KPOINT_BANDS", 0) != 0;
    HS_CUDA(cudaStreamWaitEvent(e->stream, e->ev_kup[set], 0));
    mark_build_begin(e);
    // S and H storage: k-1's downloads (enqueued in the previous iteration, download slot
    // (k-1) & 1) first
    e->wait_before_s = download_done_s(e, slot_of(k - 1));
    e->wait_before_h = download_done_h(e, slot_of(k - 1));
    try {
      enqueue_chunk(e, set ? e->whole2[0] : e->whole[0], algo, true, nullptr);
    } catch (...) {
      e->wait_before_s = e->wait_before_h = nullptr;
      e->band_final_h = false;
      throw;
    }
    e->wait_before_s = e->wait_before_h = nullptr;
    e->band_final_h = false;
    HS_CUDA(cudaEventRecord(e->ev_kbuilt[set], e->stream));
    mark_build_end(e);
    const double t_enq = trace_on() ? host_ms() : 0.0;
    if (k + 1 < nk) upload(k + 1);  // overlaps build k
    const double t_up = trace_on() ? host_ms() : 0.0;
    // k's D2H goes on the copy stream BEFORE the host unpacks an earlier k-point (another
    // download slot), so it starts as soon as build k ends instead of after the unpack
    enqueue_download(e, slot_of(k));
    if (k + 1 >= static_cast<uint64_t>(depth)) {  // overlaps build k
      const uint64_t j = k + 1 - depth;
      finish_download(e, H[j], S[j], std::chrono::steady_clock::now(), slot_of(j));
    }
    if (trace_on())
      std::fprintf(stderr, "[hsdla_b200 trace] k-point %llu: build enqueued %.2f, upload enqueued +%.2f, "
                   "previous download finished +%.2f ms\n", static_cast<unsigned long long>(k), t_enq,
                   t_up - t_enq, host_ms() - t_up);
  }
  for (uint64_t j = nk + 1 > static_cast<uint64_t>(depth) ? nk + 1 - depth : 0; j < nk; ++j)
    finish_download(e, H[j], S[j], std::chrono::steady_clock::now(), slot_of(j));
}

}  // namespace hsdla_b200
