// The path's one exchange step and the way out of the device: the sum of the partial
// H, S of the engines that share a column window (H and S are sums over
// atoms, pipeline.cpp:296-324), ownership of the reduced ranges, downloads into the
// caller's lower triangles, and per-build statistics.
//
// Reduce segments.  A build's result is reduced segment by segment: the tile-column bands
// of a banded final H contraction (band q's reduce overlaps band q+1's compute; S, computed
// first, uses the same segments and overlaps the H phases), or the whole window.  In
// SCATTER mode rank r of P owns the r-th of P equal slices of every segment (the last rank
// also the remainder): ncclReduceScatter in place (+ an ncclReduce of the remainder), so no
// GPU receives more than 1/P of H and S and every GPU downloads its own slices over its own
// PCIe link.  ROOT mode sums everything onto one rank (ncclReduce).  Engines that share one
// device (single-GPU emulation of a multi-GPU grid, tests) are summed by a deterministic
// kernel on the owner's stream instead of NCCL; ownership is identical.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "device.hpp"
#include "engine.hpp"
#include "host_pool.hpp"

namespace hsdla_b200 {

using Range = std::pair<uint64_t, uint64_t>;

static uint64_t piece_col(const hsdla_b200_engine* e, int q) {
  return std::min<uint64_t>(e->ng, static_cast<uint64_t>(e->piece_tiles[q]) * kTriBM);
}

// Global packed ranges of the reduce segments of the last build (see the file comment).
static std::vector<Range> segments(const hsdla_b200_engine* e) {
  std::vector<Range> s;
  if (e->banded) {
    for (int q = 0; q < hsdla_b200_engine::kD2hPieces; ++q)
      s.emplace_back(packed_col(e->ng, piece_col(e, q)), packed_col(e->ng, piece_col(e, q + 1)));
  } else {
    s.emplace_back(e->pk0, e->pk0 + e->npk);
  }
  return s;
}

// The slice of segment [s0, s1) that rank r of P owns after a SCATTER reduce.
static Range scatter_slice(uint64_t s0, uint64_t s1, int r, int P) {
  const uint64_t rc = (s1 - s0) / static_cast<uint64_t>(P);
  const uint64_t o0 = s0 + static_cast<uint64_t>(r) * rc;
  return {o0, r == P - 1 ? s1 : o0 + rc};
}

// The part of segment [s0, s1) this engine holds final values for.
static Range owned_part(const hsdla_b200_engine* e, uint64_t s0, uint64_t s1) {
  if (!e->reduced || e->nranks <= 1) return {s0, s1};
  if (e->red_mode == kReduceRoot) return e->rank == e->red_root ? Range{s0, s1} : Range{s1, s1};
  return scatter_slice(s0, s1, e->rank, e->nranks);
}

std::vector<Range> engine_owned(const hsdla_b200_engine* e) {
  std::vector<Range> out;
  if (!e->built) return out;
  for (const Range& sg : segments(e)) {
    const Range o = owned_part(e, sg.first, sg.second);
    if (o.second > o.first) out.push_back(o);
  }
  return out;
}

// NCCL reduce of one segment of `buf` (the engine's packed window) on its comm stream.
static void nccl_segment(hsdla_b200_engine* e, double2* buf, Range sg, int mode, int root) {
  const uint64_t len = sg.second - sg.first;
  if (!len) return;
  double2* base = buf + (sg.first - e->pk0);
  if (mode == kReduceRoot) {
    HS_NCCL(ncclReduce(base, base, 2 * len, ncclFloat64, ncclSum, root, e->comm, e->comm_stream));
    return;
  }
  const uint64_t P = static_cast<uint64_t>(e->nranks), rc = len / P, rem = len - P * rc;
  if (rc)  // in place: rank r's slice is base + r rc
    HS_NCCL(ncclReduceScatter(base, base + static_cast<uint64_t>(e->rank) * rc, 2 * rc, ncclFloat64, ncclSum,
                              e->comm, e->comm_stream));
  if (rem)
    HS_NCCL(ncclReduce(base + P * rc, base + P * rc, 2 * rem, ncclFloat64, ncclSum, e->nranks - 1, e->comm,
                       e->comm_stream));
}

// Same-device group: every owner sums its slice (or the root the whole segment) from all
// members' buffers, in rank order, after all members finished the segment (`ready`).
static void local_segment(const std::vector<hsdla_b200_engine*>& g, bool s_matrix, Range sg, int mode, int root,
                          cudaEvent_t (*ready)(hsdla_b200_engine*, int), int q) {
  const int P = static_cast<int>(g.size());
  for (int r = 0; r < P; ++r) {
    hsdla_b200_engine* o = g[r];
    Range part;
    if (mode == kReduceRoot) {
      if (r != root) continue;
      part = sg;
    } else {
      part = scatter_slice(sg.first, sg.second, r, P);
    }
    for (hsdla_b200_engine* m : g) HS_CUDA(cudaStreamWaitEvent(o->comm_stream, ready(m, q), 0));
    const uint64_t n = part.second - part.first;
    if (!n) continue;
    std::vector<const double2*> in(P);
    for (int i = 0; i < P; ++i) in[i] = (s_matrix ? g[i]->Sp : g[i]->Hp) + (part.first - g[i]->pk0);
    launch_sum_partials((s_matrix ? o->Sp : o->Hp) + (part.first - o->pk0), in.data(), P, n, o->comm_stream);
  }
}

static cudaEvent_t ev_s_ready(hsdla_b200_engine* e, int) { return e->ev_s_done; }
static cudaEvent_t ev_h_ready(hsdla_b200_engine* e, int q) { return q < 0 ? e->ev_end : e->ev_h_band[q]; }

void group_reduce(const std::vector<hsdla_b200_engine*>& g, int mode, int root) {
  if (g.empty()) return;
  const int P = static_cast<int>(g.size());
  if (mode != kReduceRoot && mode != kReduceScatter) throw Fail{HSDLA_B200_CONFIG_ERROR, "unknown reduce mode"};
  const bool nccl = g[0]->comm != nullptr;
  const int nr = nccl ? g[0]->nranks : P;
  if (root < 0 || root >= nr) throw Fail{HSDLA_B200_CONFIG_ERROR, "reduce root out of range"};
  for (hsdla_b200_engine* e : g) {
    if ((e->comm != nullptr) != nccl) throw Fail{HSDLA_B200_CONFIG_ERROR, "mixed NCCL / local reduce group"};
    if (!e->built) throw Fail{HSDLA_B200_CONFIG_ERROR, "reduce before build"};
    if (e->ng != g[0]->ng || e->c0 != g[0]->c0 || e->c1 != g[0]->c1 || e->banded != g[0]->banded)
      throw Fail{HSDLA_B200_CONFIG_ERROR, "reduce group members differ in shape / window / banding"};
    if (!nccl && e->device != g[0]->device)
      throw Fail{HSDLA_B200_CONFIG_ERROR, "engines without a communicator must share one device"};
  }
  if (!nccl) {
    if (P <= 1) return;  // a single engine holds the sum already
    for (int r = 0; r < P; ++r) {
      g[r]->nranks = P;
      g[r]->rank = r;
    }
  }
  // a group formed after its builds began: the reduce is timed from here (the builds' end)
  for (hsdla_b200_engine* e : g)
    if (!e->marks_timed) {
      HS_CUDA(cudaSetDevice(e->device));
      HS_CUDA(cudaEventRecord(e->ev_end_t, e->stream));
    }
  const std::vector<Range> segs = segments(g[0]);
  const bool banded = g[0]->banded;
  auto run = [&](bool s_matrix) {
    for (size_t q = 0; q < segs.size(); ++q) {
      const int qi = banded ? static_cast<int>(q) : -1;
      if (nccl) {
        HS_NCCL(ncclGroupStart());
        for (hsdla_b200_engine* e : g) {
          HS_CUDA(cudaSetDevice(e->device));
          HS_CUDA(cudaStreamWaitEvent(e->comm_stream, s_matrix ? e->ev_s_done : ev_h_ready(e, qi), 0));
          nccl_segment(e, s_matrix ? e->Sp : e->Hp, segs[q], mode, root);
        }
        HS_NCCL(ncclGroupEnd());
      } else {
        HS_CUDA(cudaSetDevice(g[0]->device));
        local_segment(g, s_matrix, segs[q], mode, root, s_matrix ? ev_s_ready : ev_h_ready, qi);
      }
      if (!s_matrix && banded)
        for (hsdla_b200_engine* e : g) {
          HS_CUDA(cudaSetDevice(e->device));
          HS_CUDA(cudaEventRecord(e->ev_h_red[q], e->comm_stream));
        }
    }
    if (s_matrix)
      for (hsdla_b200_engine* e : g) {
        HS_CUDA(cudaSetDevice(e->device));
        HS_CUDA(cudaEventRecord(e->ev_s_red, e->comm_stream));
      }
  };
  // S first (its partials are final after phase s: this overlaps the H phases), then H
  run(true);
  run(false);
  for (hsdla_b200_engine* e : g) {
    HS_CUDA(cudaSetDevice(e->device));
    HS_CUDA(cudaEventRecord(e->ev_reduce_end, e->comm_stream));
    HS_CUDA(cudaStreamWaitEvent(e->stream, e->ev_reduce_end, 0));
    e->red_mode = mode;
    e->red_root = root;
    e->reduced = true;
  }
  // a local group's owners read the other members' buffers on their own comm streams: no
  // member may start its next build (overwrite H, S) before every owner is done
  if (!nccl)
    for (hsdla_b200_engine* m : g)
      for (hsdla_b200_engine* o : g)
        if (m != o) HS_CUDA(cudaStreamWaitEvent(m->stream, o->ev_reduce_end, 0));
}

// Multi-process use: this process's engine is one rank of its window's communicator.
void engine_reduce(hsdla_b200_engine* e, int root) {
  if (!e->comm) return;
  group_reduce({e}, e->red_mode, root);
}

uint64_t executed_flops(uint64_t na, uint64_t nl, uint64_t ng, int arith, int algo, uint64_t rows) {
  // Real flops the GPU executes for a build.  The refined, fused and original algorithms
  // run lower-triangular contractions of 20 K N_G^2 + 24 N_A N_L^2 N_G complex-MAC flops at
  // 8 per MAC (the original's trmm on the zero upper half of L and its full gemm fold are
  // executed as the lower-only h_aa contraction); the merged one 16 K N_G^2 + 32 N_A N_L^2
  // N_G (two H segments, four per-atom products).  Plus 2 K N_G for diag_scale; the 3M
  // arithmetic executes 6 real flops per complex MAC.
  // rows: the contracted K rows (a row-balanced shard; 0: all na * nl)
  const uint64_t K = na * nl, R = rows ? rows : K;
  const uint64_t cmac8 = algo == HSDLA_B200_ALGO_REFINED_MERGED ? 16 * R * ng * ng + 32 * na * nl * nl * ng
                                                                : 20 * R * ng * ng + 24 * na * nl * nl * ng;
  return (arith == HSDLA_B200_ARITH_3M ? cmac8 / 8 * 6 : cmac8) + 2 * K * ng;
}

void flop_model(int variant, uint64_t na, uint64_t nl, uint64_t ng, uint64_t n_hpd, uint64_t* l) {
  // pipeline.cpp:336-364
  const uint64_t n_fail = na - std::min(n_hpd, na);
  std::memset(l, 0, 9 * sizeof(uint64_t));
  l[0] = 8 * na * nl * nl * ng;
  l[1] = 8 * na * nl * nl * ng;
  l[2] = 8 * na * nl * ng * ng;
  l[3] = 8 * na * nl * ng * ng;
  l[4] = 2 * na * nl * ng;
  if (variant == 0) {
    l[6] = na * (4 * nl * nl * nl / 3);
    if (n_hpd > 0) {
      l[7] = 4 * n_hpd * nl * nl * ng;
      l[3] += 4 * n_hpd * nl * ng * ng;
    }
    if (n_fail > 0) {
      l[1] += 8 * n_fail * nl * nl * ng;
      l[0] += 8 * n_fail * nl * ng * ng;
    }
  } else {
    l[1] += 8 * na * nl * nl * ng;
    l[5] = 4 * na * nl * ng * ng;
  }
  for (int i = 0; i < 8; ++i) l[8] += l[i];
}

void engine_sync(hsdla_b200_engine* e, hsdla_b200_stats* st) {
  HS_CUDA(cudaSetDevice(e->device));
  HS_CUDA(cudaStreamSynchronize(e->stream));
  HS_CUDA(cudaStreamSynchronize(e->copy_stream));
  HS_CUDA(cudaStreamSynchronize(e->comm_stream));
  for (auto& t : e->ring) harvest(e, t);
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  st->peak_device_bytes = e->device_bytes;
  // the temporaries the algorithm needs: X1 (refined, cf. pipeline.cpp:291) or X1 + X2
  st->peak_temp_bytes = (e->built && e->last_algo != HSDLA_B200_ALGO_REFINED ? 2 : 1) * e->temp_bytes;
  st->n_gpus = e->nranks;
  st->col_groups = 1;
  st->reduce_mode = e->red_mode;
  if (!e->built) return;  // nothing timed yet
  if (e->last_algo == HSDLA_B200_ALGO_ORIGINAL) {
    std::vector<int32_t> info(e->na);
    HS_CUDA(cudaMemcpy(info.data(), e->info, e->na * sizeof(int32_t), cudaMemcpyDeviceToHost));
    // the owned atoms only (a boundary atom of a row-balanced grid is factorised on two engines)
    e->n_hpd_last = static_cast<uint64_t>(std::count_if(info.begin() + e->own_a0, info.begin() + e->own_a1,
                                                        [](int32_t v) { return v < 0; }));
  } else {
    e->n_hpd_last = e->own_a1 - e->own_a0;
  }
  st->n_hpd = e->n_hpd_last;
  st->executed_flops = executed_flops(e->na, e->nl, e->ng, e->arith, e->last_algo, e->row1 - e->row0);
  // phase and device times from the launch timestamp slots (stamp.cuh): a phase op spans its
  // first kernel's start to its last kernel's end; the build spans all of its kernels
  std::vector<unsigned long long> ts(static_cast<size_t>(e->stamp_used) * kStampWords);
  if (!ts.empty()) {  // on the engine's own stream: no implicit sync with the legacy default stream
    HS_CUDA(cudaMemcpyAsync(ts.data(), e->d_stamp, ts.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            e->stream));
    HS_CUDA(cudaStreamSynchronize(e->stream));
  }
  auto span = [&](int s0, int s1) {
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int i = s0; i < s1; ++i) {
      t0 = std::min(t0, ts[static_cast<size_t>(i) * kStampWords]);
      t1 = std::max(t1, ts[static_cast<size_t>(i) * kStampWords + 1]);
    }
    return t1 > t0 ? static_cast<double>(t1 - t0) * 1e-9 : 0.0;
  };
  for (const OpTime& op : e->ops) st->phase_seconds[op.phase] += span(op.s0, op.s1);
  // (the reduce tail after the build's end; a banded reduce can finish with the build)
  st->reduce_seconds = e->reduced ? std::max(0.0, ev_ms(e->ev_end_t, e->ev_reduce_end) * 1e-3) : 0.0;
  st->device_seconds = e->reduced && e->marks_timed ? ev_ms(e->ev_begin, e->ev_reduce_end) * 1e-3
                                                    : span(0, e->stamp_used) + st->reduce_seconds;
  if (e->uploaded_streamed) st->h2d_seconds = ev_ms(e->ev_up0, e->ev_up1) * 1e-3;
  st->kernel_launches = e->launches;
}

// One download slot: its pinned stage, its copy-stream events and its record.
struct DlSlot {
  double2* stage;
  cudaEvent_t ev_s;
  cudaEvent_t* ev_h;
  Download& d;
};

// Slot 0's stage is allocated on first use; slots 1 and 2 (k-point batches) get their stage
// and events all-or-nothing on first use.
static DlSlot dl_slot(hsdla_b200_engine* e, int slot) {
  if (slot == 0) {
    if (!e->host_stage)
      HS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&e->host_stage), 2 * e->cap_pk * sizeof(double2)));
    return {e->host_stage, e->ev_dl_s, e->ev_dl_h, e->dl};
  }
  const int x = slot - 1;
  if (!e->host_stage_x[x]) {
    double2* st = nullptr;
    cudaEvent_t ev[1 + hsdla_b200_engine::kD2hPieces] = {};
    try {
      HS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&st), 2 * e->cap_pk * sizeof(double2)));
      for (cudaEvent_t& ev1 : ev) HS_CUDA(cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming));
    } catch (...) {
      if (st) cudaFreeHost(st);
      for (cudaEvent_t ev1 : ev)
        if (ev1) cudaEventDestroy(ev1);
      throw;
    }
    e->ev_dlx_s[x] = ev[0];
    for (int q = 0; q < hsdla_b200_engine::kD2hPieces; ++q) e->ev_dlx_h[x][q] = ev[1 + q];
    e->host_stage_x[x] = st;
  }
  return {e->host_stage_x[x], e->ev_dlx_s[x], e->ev_dlx_h[x], e->dlx[x]};
}

cudaEvent_t download_done_s(hsdla_b200_engine* e, int slot) { return slot ? e->ev_dlx_s[slot - 1] : e->ev_dl_s; }
cudaEvent_t download_done_h(hsdla_b200_engine* e, int slot) {
  return (slot ? e->ev_dlx_h[slot - 1] : e->ev_dl_h)[hsdla_b200_engine::kD2hPieces - 1];
}

// Enqueue the packed-triangle D2H of the ranges this engine owns on the copy stream: S
// (after phase s / its reduce), then H in kD2hPieces column pieces (after band q / its
// reduce when banded, else after the build / its reduce), each piece's event recorded so
// the host unpacks piece q while q+1 is on the wire.  Every event is recorded every time
// (the next k-point's build waits on the last one).
void enqueue_download(hsdla_b200_engine* e, int slot) {
  HS_CUDA(cudaSetDevice(e->device));
  const DlSlot sl = dl_slot(e, slot);
  Download& d = sl.d;
  d.ng = e->ng;
  d.pk0 = e->pk0;
  d.seq.clear();
  cudaStream_t cs = e->copy_stream;
  trace_mark(e, cs, "dl_enq");
  const std::vector<Range> own = engine_owned(e);
  HS_CUDA(cudaStreamWaitEvent(cs, e->reduced ? e->ev_s_red : e->ev_s_done, 0));
  for (const Range& o : own) {
    HS_CUDA(cudaMemcpyAsync(sl.stage + e->cap_pk + (o.first - e->pk0), e->Sp + (o.first - e->pk0),
                            (o.second - o.first) * sizeof(double2), cudaMemcpyDeviceToHost, cs));
    d.seq.push_back({0, o.first, o.second, sl.ev_s});
  }
  HS_CUDA(cudaEventRecord(sl.ev_s, cs));
  trace_mark(e, cs, "dl_s");
  if (!e->banded) HS_CUDA(cudaStreamWaitEvent(cs, e->reduced ? e->ev_reduce_end : e->ev_end, 0));
  for (int q = 0; q < hsdla_b200_engine::kD2hPieces; ++q) {
    // banded: piece q is final once band q is computed (one engine) or reduced (group)
    if (e->banded) HS_CUDA(cudaStreamWaitEvent(cs, e->reduced ? e->ev_h_red[q] : e->ev_h_band[q], 0));
    const uint64_t p0 = packed_col(e->ng, piece_col(e, q)), p1 = packed_col(e->ng, piece_col(e, q + 1));
    for (const Range& o : own) {
      const uint64_t b0 = std::max(p0, o.first), b1 = std::min(p1, o.second);
      if (b1 <= b0) continue;
      HS_CUDA(cudaMemcpyAsync(sl.stage + (b0 - e->pk0), e->Hp + (b0 - e->pk0), (b1 - b0) * sizeof(double2),
                              cudaMemcpyDeviceToHost, cs));
      d.seq.push_back({1, b0, b1, sl.ev_h[q]});
    }
    HS_CUDA(cudaEventRecord(sl.ev_h[q], cs));
    if (trace_on()) trace_mark(e, cs, "dl_h" + std::to_string(q));
  }
  d.pending = true;
}

// Unpack S as soon as its bytes land (H may still be computing), then H piece by piece.
void finish_download(hsdla_b200_engine* e, double* H, double* S, std::chrono::steady_clock::time_point t0,
                     int slot) {
  const DlSlot sl = dl_slot(e, slot);
  Download& d = sl.d;
  if (!d.pending) return;
  auto ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
  std::string tr;
  auto mark = [&](const char* what) {
    if (trace_on()) tr += std::string(" ") + what + "=" + std::to_string(ms()).substr(0, 6);
  };
  d.pending = false;
  // a stage that fits the cores' L2s (16 x 2 MB on the measured host) stays cached after the
  // unpack reads it unless demoted (host_pool.cpp); HSDLA_B200_STAGE_DEMOTE_MB overrides
  static const double demote_mb = env_double("HSDLA_B200_STAGE_DEMOTE_MB", 48.0);
  uint64_t stage_elems = 0;
  for (const DlPiece& p : d.seq) stage_elems += p.b1 - p.b0;
  const bool release = static_cast<double>(stage_elems) * sizeof(double2) < demote_mb * (1 << 20);
  // Pieces in landing order; consecutive pieces of the same matrix that are contiguous (either
  // direction) and have all landed by the time the first is waited for are unpacked in ONE
  // pass over the host pool (an unbanded build's eight H pieces land together: one 16-thread
  // unpack instead of eight small ones)
  auto landed = [](cudaEvent_t ev) {
    const cudaError_t r = cudaEventQuery(ev);
    if (r == cudaSuccess) return true;
    if (r != cudaErrorNotReady) HS_CUDA(r);
    return false;
  };
  for (size_t i = 0; i < d.seq.size();) {
    HS_CUDA(cudaEventSynchronize(d.seq[i].ready));
    mark(d.seq[i].h ? "h_landed" : "s_landed");
    uint64_t lo = d.seq[i].b0, hi = d.seq[i].b1;
    size_t j = i + 1;
    for (; j < d.seq.size(); ++j) {
      const DlPiece& q = d.seq[j];
      if (q.h != d.seq[i].h || !(q.ready == d.seq[i].ready || landed(q.ready))) break;
      if (q.b0 == hi)
        hi = q.b1;
      else if (q.b1 == lo)
        lo = q.b0;
      else
        break;
    }
    double* dst = d.seq[i].h ? H : S;
    if (dst)
      unpack_range(sl.stage + (d.seq[i].h ? 0 : e->cap_pk) + (lo - d.pk0), reinterpret_cast<double2*>(dst), d.ng,
                   lo, hi, release);
    i = j;
  }
  HS_CUDA(cudaEventSynchronize(sl.ev_h[hsdla_b200_engine::kD2hPieces - 1]));
  mark("h_unpacked");
  if (trace_on()) {
    std::fprintf(stderr, "[hsdla_b200 trace] download (ms since call start):%s\n", tr.c_str());
    if (!e->tr_marks.empty()) {
      // (a k-point batch has the next build's marks in flight by now: the trace waits for
      // them, which serialises the batch while tracing)
      std::string dv;
      for (auto& m : e->tr_marks) {
        HS_CUDA(cudaEventSynchronize(m.second));
        dv += " " + m.first + "=" + std::to_string(ev_ms(e->tr_marks[0].second, m.second)).substr(0, 5);
      }
      std::fprintf(stderr, "[hsdla_b200 trace] device (ms since first mark):%s\n", dv.c_str());
      e->tr_marks.clear();
    }
  }
}

void engine_download(hsdla_b200_engine* e, double* H, double* S) {
  HS_CUDA(cudaSetDevice(e->device));
  if (!e->built) throw Fail{HSDLA_B200_CONFIG_ERROR, "download before build"};
  enqueue_download(e);
  finish_download(e, H, S);
}

}  // namespace hsdla_b200
