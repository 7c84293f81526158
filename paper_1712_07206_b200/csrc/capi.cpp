// The C-ABI of the drop-in (include/hsdla_b200.h): the one-shot build_hs / build_hs_file /
// k-point calls over a cached grid of engines, and the engine-level API that multi-process
// callers (one process per GPU, e.g. torchrun) drive themselves.
//
// Multi-GPU grid of the one-shot calls: n_gpus = col_groups x atom_ranks engines.  Engine
// (g, r) holds row shard r (shard_rows: an even split of the K rows) and column window g (equal-work tile-column
// windows) of H and S.  The atom ranks of a window sum their partials (group_reduce:
// NCCL over the window's GPUs, or a sum kernel for engines that share a device); windows
// never exchange data.  col_groups = 1 is plain atom sharding with H, S replicated per GPU;
// larger col_groups divide each GPU's H, S storage (2-D tiling, chosen when the per-GPU
// memory estimate exceeds the budget).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
#include <tuple>

#include "device.hpp"
#include "engine.hpp"
#include "hsdl_file.hpp"

namespace hsdla_b200 {

thread_local std::string g_last_error;

// ---------------------------------------------------------------------------
// the one-shot drop-in: cached engine grids, NCCL communicators, reduce, download
// ---------------------------------------------------------------------------
struct EngineSet {
  int pc = 1, pa = 1;                                // column windows x atom ranks
  std::vector<hsdla_b200_engine*> engines;           // engine (g, r) at g * pa + r
  std::vector<uint64_t> atom0;                       // first atom of each engine
  std::vector<std::vector<hsdla_b200_engine*>> groups;  // per window: its atom ranks
  uint64_t ng = 0;
  ~EngineSet() {
    for (auto* e : engines) {
      engine_free(e);
      delete e;
    }
  }
};

static std::mutex g_cache_mu;
// one grid at a time keeps HBM free for the caller: key (devices, n_atoms, n_l, col_groups)
static std::map<std::tuple<std::vector<int>, uint64_t, uint64_t, int>, std::unique_ptr<EngineSet>> g_cache;
// NCCL communicators per (window index, device list), independent of the problem shape:
// a shape change re-creates engines but never re-initialises NCCL
static std::map<std::pair<int, std::vector<int>>, std::vector<ncclComm_t>> g_comms;

static void release_comms() {
  for (auto& kv : g_comms)
    for (ncclComm_t c : kv.second) ncclCommDestroy(c);
  g_comms.clear();
}

// Contiguous, count-balanced atom ranges.
static std::vector<uint64_t> shard_atoms(uint64_t na, int parts) {
  std::vector<uint64_t> b(parts + 1);
  for (int r = 0; r <= parts; ++r) b[r] = na * r / parts;
  return b;
}

// Row-balanced shards: the K = na nl rows split evenly (the H/S contractions, ~all of the
// work, then take equal time on every GPU: 108 atoms over 8 GPUs is 1633-1634 rows each instead
// of 14 vs 13 atoms).  Shard r holds the atoms its rows touch: {atom_begin, n_atoms_local,
// row0, row1} with the row range local to its first atom.
struct RowShard {
  uint64_t a0, na, row0, row1;
};
static std::vector<RowShard> shard_rows(uint64_t na, uint64_t nl, int parts) {
  const uint64_t K = na * nl;
  if (static_cast<uint64_t>(parts) > K) throw Fail{HSDLA_B200_CONFIG_ERROR, "more shards than K rows"};
  std::vector<RowShard> out(parts);
  for (int r = 0; r < parts; ++r) {
    const uint64_t k0 = K * r / parts, k1 = K * (r + 1) / parts;
    const uint64_t a0 = k0 / nl, a1 = (k1 + nl - 1) / nl;
    out[r] = {a0, a1 - a0, k0 - a0 * nl, k1 - a0 * nl};
  }
  return out;
}

// Column boundaries of `parts` windows of (about) equal lower-triangle work; interior
// boundaries are multiples of 64 (the tile width), the last is ng.
static std::vector<uint64_t> col_windows(uint64_t ng, int parts) {
  const uint64_t T = (ng + kTriBM - 1) / kTriBM;
  if (static_cast<uint64_t>(parts) > T) throw Fail{HSDLA_B200_CONFIG_ERROR, "more column windows than tile columns"};
  const double total = static_cast<double>(T) * (T + 1) / 2;
  std::vector<uint64_t> w{0};
  uint64_t tj = 0;
  double acc = 0;
  for (int g = 1; g < parts; ++g) {
    const double target = total * g / parts;
    while (tj < T && acc + (T - tj) <= target) acc += static_cast<double>(T - tj++);
    // at least one tile column per window
    tj = std::max<uint64_t>(tj, w.back() / kTriBM + 1);
    tj = std::min<uint64_t>(tj, T - (parts - g));
    w.push_back(tj * kTriBM);
  }
  w.push_back(ng);
  return w;
}

// Device bytes of the largest engine of a pc x pa grid (window 0 holds every operand
// column; the merged algorithm's four K x N_G stacks, its packed H, S and the operator blocks).
static double grid_bytes(uint64_t na, uint64_t nl, uint64_t ng, int pc, int pa) {
  // a row-balanced shard holds up to one atom more than na / pa (the atoms its rows touch)
  const double na_r = std::min<double>(na, std::ceil(static_cast<double>(na) / pa) + (pa > 1)), K = na_r * nl;
  const double pk = static_cast<double>(ng) * (ng + 1) / 2 / pc;
  return 16.0 * (4.0 * K * ng + 2.0 * pk * 1.1 + 6.0 * na_r * nl * nl);
}

static int choose_col_groups(const hsdla_b200_options* o, const std::vector<int>& devs, uint64_t na, uint64_t nl,
                             uint64_t ng) {
  const int P = static_cast<int>(devs.size());
  if (o && o->col_groups > 0) {
    if (P % o->col_groups != 0) throw Fail{HSDLA_B200_CONFIG_ERROR, "col_groups must divide n_gpus"};
    return o->col_groups;
  }
  if (P == 1) return 1;
  double budget = o && o->mem_budget_gb > 0 ? o->mem_budget_gb * 1e9 : 0.0;
  if (budget <= 0) {
    budget = 1e300;
    for (int d : std::set<int>(devs.begin(), devs.end())) {
      size_t fr = 0, tot = 0;
      HS_CUDA(cudaSetDevice(d));
      HS_CUDA(cudaMemGetInfo(&fr, &tot));
      // engines sharing a device (emulation) share its memory
      const int sharing = static_cast<int>(std::count(devs.begin(), devs.end(), d));
      budget = std::min(budget, 0.9 * static_cast<double>(fr) / sharing);
    }
  }
  int best = 1;
  double best_b = 1e300;
  for (int pc = 1; pc <= P; ++pc) {
    if (P % pc) continue;
    if (static_cast<uint64_t>(P / pc) > na) continue;
    const double b = grid_bytes(na, nl, ng, pc, P / pc);
    if (b <= budget) return pc;  // the least 2-D tiling that fits
    if (b < best_b) {
      best_b = b;
      best = pc;
    }
  }
  return best;  // nothing fits: the smallest footprint (allocation reports SizingError if it fails)
}

static EngineSet* get_engines(const std::vector<int>& devs, uint64_t na, uint64_t nl, uint64_t ng, int pc,
                              uint64_t ng_capacity = 0) {
  const int P = static_cast<int>(devs.size()), pa = P / pc;
  auto key = std::make_tuple(devs, na, nl, pc);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    EngineSet* set = it->second.get();
    if (pc == 1 && ng_capacity <= set->engines[0]->cap_cols) {
      bool ok = true;
      for (auto* e : set->engines) ok = ok && engine_reshape(e, ng);
      if (ok) {
        set->ng = ng;
        return set;
      }
    } else if (set->ng == ng) {
      return set;
    }
  }
  g_cache.clear();  // one grid at a time keeps HBM free for the caller
  if (static_cast<uint64_t>(pa) > na) throw Fail{HSDLA_B200_CONFIG_ERROR, "more GPUs than atoms"};
  const auto rs = shard_rows(na, nl, pa);
  const auto cw = col_windows(ng, pc);
  auto make = [&](uint64_t cap) {
    auto set = std::make_unique<EngineSet>();
    set->pc = pc;
    set->pa = pa;
    set->ng = ng;
    for (int g = 0; g < pc; ++g) {
      set->groups.emplace_back();
      for (int r = 0; r < pa; ++r) {
        ShardSpec sp;
        sp.na = rs[r].na;
        sp.row0 = rs[r].row0;
        sp.row1 = rs[r].row1;
        sp.nl = nl;
        sp.ng = ng;
        sp.c0 = cw[g];
        sp.c1 = cw[g + 1];
        sp.ng_capacity = cap;
        hsdla_b200_engine* e = engine_create(devs[g * pa + r], sp);
        set->engines.push_back(e);
        e->rank = r;
        e->nranks = pa;
        set->atom0.push_back(rs[r].a0);
        set->groups.back().push_back(e);
      }
    }
    return set;
  };
  // whole-window grids get 5 % of N_G headroom: a k-point loop whose N_G(k) varies by a few
  // per cent re-targets the cached engines instead of reallocating them (exact sizes when the
  // headroom does not fit in HBM)
  const uint64_t exact = std::max(ng_capacity, ng), cap = pc == 1 ? std::max(exact, ng + ng / 20) : ng;
  std::unique_ptr<EngineSet> set;
  try {
    set = make(cap);
  } catch (const Fail& f) {
    if (f.code != HSDLA_B200_SIZING_ERROR || cap == exact) throw;
    set = make(exact);
  }
  // per window group: NCCL over distinct devices, or the local sum kernel on one device
  for (int g = 0; g < pc && pa > 1; ++g) {
    std::vector<int> gd(devs.begin() + g * pa, devs.begin() + (g + 1) * pa);
    const std::set<int> uniq(gd.begin(), gd.end());
    if (uniq.size() == 1) {
      for (auto* e : set->groups[g]) e->local_group = set->groups[g];
      continue;
    }
    if (static_cast<int>(uniq.size()) != pa)
      throw Fail{HSDLA_B200_CONFIG_ERROR,
                 "the GPUs of a column window must be all distinct (NCCL) or all one device (emulation)"};
    auto& comms = g_comms[{g, gd}];
    if (comms.empty()) {
      comms.resize(pa);
      HS_NCCL(ncclCommInitAll(comms.data(), pa, gd.data()));
    }
    for (int r = 0; r < pa; ++r) {
      set->groups[g][r]->comm = comms[r];
      set->groups[g][r]->comm_owned = false;
    }
  }
  EngineSet* raw = set.get();
  g_cache.emplace(key, std::move(set));
  return raw;
}

static std::vector<int> devices_of(const hsdla_b200_options* o) {
  const int P = o && o->n_gpus > 1 ? o->n_gpus : 1;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    (void)cudaGetLastError();
    throw Fail{HSDLA_B200_CONFIG_ERROR, "no CUDA device visible (the B200 path has no CPU fallback)"};
  }
  std::vector<int> devs(P);
  for (int r = 0; r < P; ++r) devs[r] = (o && o->device_ids) ? o->device_ids[r] : r;
  for (int d : devs)
    if (d < 0 || d >= ndev) throw Fail{HSDLA_B200_CONFIG_ERROR, "device id out of range"};
  return devs;
}

static constexpr int kKnownFlags = HSDLA_B200_FLAG_ARITH_4M | HSDLA_B200_FLAG_REDUCE_ROOT;

// Run fn(i) for i in [0, n) on n host threads (inline for n == 1), rethrowing the first failure.
template <class F>
static void on_threads(int n, F&& fn) {
  std::vector<Fail> errs(n);
  std::vector<char> bad(n, 0);
  auto run = [&](int i) {
    try {
      fn(i);
    } catch (const Fail& f) {
      errs[i] = f;
      bad[i] = 1;
    } catch (const std::exception& x) {
      errs[i] = Fail{HSDLA_B200_CUDA_ERROR, x.what()};
      bad[i] = 1;
    }
  };
  if (n == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (int i = 0; i < n; ++i) th.emplace_back(run, i);
    for (auto& t : th) t.join();
  }
  for (int i = 0; i < n; ++i)
    if (bad[i]) throw errs[i];
}

// The one-shot drop-in around a per-engine "start" (upload/load + enqueue build,
// returning host seconds spent loading): device selection, engine grid, reduce,
// overlapped per-GPU downloads, stats.
template <class Start>
static void one_shot(const hsdla_b200_options* o, uint64_t na, uint64_t nl, uint64_t ng, double* H, double* S,
                     hsdla_b200_stats* st, std::chrono::steady_clock::time_point t0, Start&& start) {
  const int algo = o ? o->algo : HSDLA_B200_ALGO_REFINED_MERGED;
  if (!valid_algo(algo)) throw Fail{HSDLA_B200_CONFIG_ERROR, "unknown algo " + std::to_string(algo)};
  if (o && (o->flags & ~kKnownFlags)) throw Fail{HSDLA_B200_CONFIG_ERROR, "unknown option flags"};
  if (o && o->col_groups < 0) throw Fail{HSDLA_B200_CONFIG_ERROR, "col_groups must be >= 0"};
  const int arith = o && (o->flags & HSDLA_B200_FLAG_ARITH_4M) ? HSDLA_B200_ARITH_4M : HSDLA_B200_ARITH_3M;
  const int mode = o && (o->flags & HSDLA_B200_FLAG_REDUCE_ROOT) ? kReduceRoot : kReduceScatter;
  const std::vector<int> devs = devices_of(o);
  const int P = static_cast<int>(devs.size());
  if (trace_on())
    std::fprintf(stderr, "[hsdla_b200 trace] call start at %.3f ms (host clock)\n",
                 std::chrono::duration<double, std::milli>(t0.time_since_epoch()).count());
  std::lock_guard<std::mutex> lk(g_cache_mu);
  const int pc = choose_col_groups(o, devs, na, nl, ng);
  EngineSet* set = get_engines(devs, na, nl, ng, pc);
  // One host thread per engine (a file-backed start reads that engine's shard on the host).
  // Every final H contraction runs band by band: the download (one GPU) or the reduce of
  // band q overlaps the compute of band q+1.
  std::vector<double> load(P, 0.0);
  on_threads(P, [&](int i) {
    hsdla_b200_engine* e = set->engines[i];
    e->band_final_h = true;
    e->arith = arith;
    try {
      load[i] = start(e, set->atom0[i], algo);
    } catch (...) {
      e->band_final_h = false;
      throw;
    }
    e->band_final_h = false;
  });
  const double load_s = *std::max_element(load.begin(), load.end());
  if (set->pa > 1)
    for (auto& g : set->groups) group_reduce(g, mode, 0);
  // every engine downloads the ranges it owns into the caller's H, S (disjoint), each over its
  // own PCIe link and host thread
  const auto t_d = std::chrono::steady_clock::now();
  if (trace_on())
    std::fprintf(stderr, "[hsdla_b200 trace] enqueued at %.3f ms since call start\n",
                 std::chrono::duration<double, std::milli>(t_d - t0).count());
  on_threads(P, [&](int i) {
    hsdla_b200_engine* e = set->engines[i];
    HS_CUDA(cudaSetDevice(e->device));
    enqueue_download(e);
    finish_download(e, H, S, t0);
  });
  const double d2h = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_d).count();
  hsdla_b200_stats local{};
  double maxph[HSDLA_B200_N_PHASES] = {};
  double dev_s = 0, red_s = 0, h2d = 0;
  int launches = 0;
  uint64_t n_hpd = 0, peak_dev = 0, peak_tmp = 0;
  for (int i = 0; i < P; ++i) {
    engine_sync(set->engines[i], &local);
    if (i < set->pa) n_hpd += local.n_hpd;  // window 0's atom ranks cover every atom once
    for (int k = 0; k < HSDLA_B200_N_PHASES; ++k) maxph[k] = std::max(maxph[k], local.phase_seconds[k]);
    dev_s = std::max(dev_s, local.device_seconds);
    red_s = std::max(red_s, local.reduce_seconds);
    h2d = std::max(h2d, local.h2d_seconds);
    launches += local.kernel_launches;
    peak_dev = std::max(peak_dev, local.peak_device_bytes);
    peak_tmp = std::max(peak_tmp, local.peak_temp_bytes);
  }
  if (st) {
    std::memcpy(st->phase_seconds, maxph, sizeof(maxph));
    st->h2d_seconds = std::max(h2d, load_s);
    st->device_seconds = dev_s;
    st->reduce_seconds = red_s;
    st->d2h_seconds = d2h;
    // ledger == pipeline::flop_model(p, variant) with the potrf outcome of this build
    flop_model(algo == HSDLA_B200_ALGO_ORIGINAL ? 0 : 1, na, nl, ng, n_hpd, st->ledger);
    st->executed_flops = executed_flops(na, nl, ng, arith, algo);
    st->n_hpd = n_hpd;
    st->peak_device_bytes = peak_dev;
    st->peak_temp_bytes = peak_tmp;
    st->n_gpus = P;
    st->kernel_launches = launches;
    st->col_groups = set->pc;
    st->reduce_mode = mode;
    st->total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
}

}  // namespace hsdla_b200

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace hsdla_b200;

extern "C" {

const char* hsdla_b200_last_error(void) { return g_last_error.c_str(); }

int hsdla_b200_device_count(int* count) {
  return guarded([&] {
    if (!count) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null count"};
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

int hsdla_b200_flop_model(int variant, uint64_t na, uint64_t nl, uint64_t ng, uint64_t n_hpd, uint64_t ledger[9]) {
  return guarded([&] {
    if (!ledger) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null ledger"};
    flop_model(variant, na, nl, ng, n_hpd, ledger);
  });
}

int hsdla_b200_potrf(int device, uint64_t nb, uint64_t nl, const double* T, double* L, int64_t* pivot) {
  return guarded([&] {
    if (!T || !L || !pivot) throw Fail{HSDLA_B200_DIMENSION_ERROR, "potrf: null pointer"};
    if (nb < 1 || nl < 1 || nl > 4096) throw Fail{HSDLA_B200_DIMENSION_ERROR, "potrf: need n_blocks >= 1, 1 <= n_l <= 4096"};
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
      (void)cudaGetLastError();
      throw Fail{HSDLA_B200_CONFIG_ERROR, "no such CUDA device (the B200 path has no CPU fallback)"};
    }
    HS_CUDA(cudaSetDevice(device));
    const size_t bytes = nb * nl * nl * sizeof(double2);
    struct Buf {
      void* p = nullptr;
      ~Buf() {
        if (p) cudaFree(p);
      }
    } dT, dL, dI;
    HS_CUDA(cudaMalloc(&dT.p, bytes));
    HS_CUDA(cudaMalloc(&dL.p, bytes));
    HS_CUDA(cudaMalloc(&dI.p, nb * sizeof(int32_t)));
    HS_CUDA(cudaMemcpy(dT.p, T, bytes, cudaMemcpyHostToDevice));
    launch_potrf_batched(static_cast<const double2*>(dT.p), static_cast<double2*>(dL.p), static_cast<int32_t*>(dI.p),
                         static_cast<int>(nl), nb, nullptr, 0);
    std::vector<int32_t> info(nb);
    HS_CUDA(cudaMemcpy(L, dL.p, bytes, cudaMemcpyDeviceToHost));
    HS_CUDA(cudaMemcpy(info.data(), dI.p, nb * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (uint64_t b = 0; b < nb; ++b) pivot[b] = info[b];
  });
}

int hsdla_b200_shard_atoms(uint64_t n_atoms, int parts, uint64_t* bounds) {
  return guarded([&] {
    if (!bounds || parts < 1) throw Fail{HSDLA_B200_CONFIG_ERROR, "shard_atoms: parts must be >= 1"};
    if (static_cast<uint64_t>(parts) > n_atoms) throw Fail{HSDLA_B200_CONFIG_ERROR, "more GPUs than atoms"};
    const auto b = shard_atoms(n_atoms, parts);
    std::copy(b.begin(), b.end(), bounds);
  });
}

int hsdla_b200_host_register(void* ptr, size_t bytes) {
  return guarded([&] { HS_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable)); });
}
int hsdla_b200_host_unregister(void* ptr) {
  return guarded([&] { HS_CUDA(cudaHostUnregister(ptr)); });
}
int hsdla_b200_release_cache(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.clear();
    release_comms();
    // the kernel layer's cached temporaries (keep_pool_cached)
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
      (void)cudaGetLastError();
      return;
    }
    for (int d = 0; d < ndev; ++d) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
        int cur = 0;
        (void)cudaGetDevice(&cur);
        (void)cudaSetDevice(d);
        (void)cudaDeviceSynchronize();
        (void)cudaMemPoolTrimTo(pool, 0);
        (void)cudaSetDevice(cur);
      }
    }
    (void)cudaGetLastError();
  });
}

int hsdla_b200_engine_create(int device, uint64_t na, uint64_t nl, uint64_t ng, hsdla_b200_engine** out) {
  return guarded([&] {
    if (!out) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null out"};
    ShardSpec sp;
    sp.na = na;
    sp.nl = nl;
    sp.ng = ng;
    *out = engine_create(device, sp);
  });
}
int hsdla_b200_shard_rows(uint64_t n_atoms, uint64_t n_l, int parts, uint64_t* shards) {
  return guarded([&] {
    if (!shards || parts < 1 || n_l < 1) throw Fail{HSDLA_B200_CONFIG_ERROR, "shard_rows: parts and n_l must be >= 1"};
    if (static_cast<uint64_t>(parts) > n_atoms) throw Fail{HSDLA_B200_CONFIG_ERROR, "more GPUs than atoms"};
    const auto rs = shard_rows(n_atoms, n_l, parts);
    for (int r = 0; r < parts; ++r) {
      shards[4 * r] = rs[r].a0;
      shards[4 * r + 1] = rs[r].na;
      shards[4 * r + 2] = rs[r].row0;
      shards[4 * r + 3] = rs[r].row1;
    }
  });
}
int hsdla_b200_engine_create_shard(int device, const hsdla_b200_shard* s, hsdla_b200_engine** out) {
  return guarded([&] {
    if (!out || !s) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null shard / out"};
    ShardSpec sp;
    sp.na = s->n_atoms_local;
    sp.nl = s->n_l;
    sp.ng = s->n_g;
    sp.c0 = s->col_begin;
    sp.c1 = s->col_end;
    sp.ng_capacity = s->n_g_capacity;
    sp.row0 = s->row_begin;
    sp.row1 = s->row_end;
    if (sp.ng_capacity && sp.ng_capacity < sp.ng) throw Fail{HSDLA_B200_CONFIG_ERROR, "n_g_capacity < n_g"};
    *out = engine_create(device, sp);
  });
}
int hsdla_b200_engine_reshape(hsdla_b200_engine* e, uint64_t ng) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    if (!(e->c0 == 0 && e->c1 == e->ng)) throw Fail{HSDLA_B200_CONFIG_ERROR, "reshape needs a whole-window engine"};
    if (!engine_reshape(e, ng)) throw Fail{HSDLA_B200_SIZING_ERROR, "n_g exceeds the engine capacity"};
  });
}
int hsdla_b200_engine_destroy(hsdla_b200_engine* e) {
  return guarded([&] {
    if (!e) return;
    engine_free(e);
    delete e;
  });
}
int hsdla_b200_engine_upload(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_upload(e, p, a0);
  });
}
int hsdla_b200_engine_fill_synthetic(hsdla_b200_engine* e, uint64_t seed) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_fill_synthetic(e, seed);
  });
}
int hsdla_b200_engine_set_arith(hsdla_b200_engine* e, int arith) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    if (arith != HSDLA_B200_ARITH_3M && arith != HSDLA_B200_ARITH_4M)
      throw Fail{HSDLA_B200_CONFIG_ERROR, "arith must be HSDLA_B200_ARITH_3M or _4M"};
    e->arith = arith;
  });
}
int hsdla_b200_engine_set_download_overlap(hsdla_b200_engine* e, int on) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    e->overlap_dl = on != 0;
    if (!on) e->band_final_h = false;
  });
}
int hsdla_b200_set_default_arith(int arith) {
  return guarded([&] {
    if (arith != HSDLA_B200_ARITH_3M && arith != HSDLA_B200_ARITH_4M)
      throw Fail{HSDLA_B200_CONFIG_ERROR, "arith must be HSDLA_B200_ARITH_3M or _4M"};
    g_default_arith.store(arith);
  });
}
int hsdla_b200_engine_build(hsdla_b200_engine* e, int algo) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_build(e, algo);
  });
}
int hsdla_b200_engine_build_streamed(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0, int algo) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_build_streamed(e, p, a0, algo);
  });
}
int hsdla_b200_engine_reduce(hsdla_b200_engine* e, int root) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_reduce(e, root);
  });
}
int hsdla_b200_engine_set_reduce_mode(hsdla_b200_engine* e, int mode) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    if (mode != HSDLA_B200_REDUCE_ROOT && mode != HSDLA_B200_REDUCE_SCATTER)
      throw Fail{HSDLA_B200_CONFIG_ERROR, "mode must be HSDLA_B200_REDUCE_ROOT or _SCATTER"};
    e->red_mode = mode;
  });
}
int hsdla_b200_group_reduce(hsdla_b200_engine* const* engines, int n, int mode, int root) {
  return guarded([&] {
    if (!engines || n < 1) throw Fail{HSDLA_B200_CONFIG_ERROR, "null / empty engine group"};
    std::vector<hsdla_b200_engine*> g(engines, engines + n);
    for (auto* e : g)
      if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    group_reduce(g, mode, root);
  });
}
int hsdla_b200_engine_owned(hsdla_b200_engine* e, uint64_t* ranges, uint64_t max, uint64_t* n) {
  return guarded([&] {
    if (!e || !n) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine / count"};
    const auto own = engine_owned(e);
    *n = own.size();
    for (uint64_t i = 0; i < std::min<uint64_t>(max, own.size()) && ranges; ++i) {
      ranges[2 * i] = own[i].first;
      ranges[2 * i + 1] = own[i].second;
    }
  });
}
int hsdla_b200_engine_sync(hsdla_b200_engine* e, hsdla_b200_stats* st) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_sync(e, st);
  });
}
int hsdla_b200_engine_download(hsdla_b200_engine* e, double* H, double* S) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_download(e, H, S);
  });
}
int hsdla_b200_engine_device_results(hsdla_b200_engine* e, void** Hp, void** Sp) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    if (Hp) *Hp = e->Hp;
    if (Sp) *Sp = e->Sp;
  });
}
int hsdla_b200_engine_stream(hsdla_b200_engine* e, void** stream) {
  return guarded([&] {
    if (!e || !stream) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    *stream = e->stream;
  });
}
int hsdla_b200_nccl_unique_id(void* id128) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    if (!id128) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null id"};
    ncclUniqueId id;
    HS_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
  });
}
int hsdla_b200_engine_set_comm(hsdla_b200_engine* e, const void* id128, int nranks, int rank) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Fail{HSDLA_B200_CONFIG_ERROR, "bad rank"};
    HS_CUDA(cudaSetDevice(e->device));
    if (e->comm && e->comm_owned) ncclCommDestroy(e->comm);
    e->comm = nullptr;
    e->comm_owned = true;
    e->nranks = nranks;
    e->rank = rank;
    if (!id128) {
      if (nranks > 1) throw Fail{HSDLA_B200_CONFIG_ERROR, "null NCCL id"};
      return;  // single rank without a communicator: reduce is a no-op
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    HS_NCCL(ncclCommInitRank(&e->comm, nranks, id, rank));
  });
}
int hsdla_b200_engine_kernel_times(hsdla_b200_engine* e, int reset, double* ms_s, double* ms_h, uint64_t* flops_s,
                                   uint64_t* flops_h, uint64_t* n_builds) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    HS_CUDA(cudaSetDevice(e->device));
    HS_CUDA(cudaStreamSynchronize(e->stream));
    for (auto& t : e->ring) harvest(e, t);
    const double n = static_cast<double>(std::max<uint64_t>(e->timed_builds, 1));
    if (ms_s) *ms_s = e->sum_s_ms / n;
    if (ms_h) *ms_h = e->sum_h_ms / n;
    // S: herk(A) + herk(UB), ledger 2 x 4 K N_G^2 (the window's share for a column window)
    if (flops_s) *flops_s = static_cast<uint64_t>(static_cast<double>(e->sum_flops_s) / n);
    if (flops_h) *flops_h = static_cast<uint64_t>(static_cast<double>(e->sum_flops_h) / n);
    if (n_builds) *n_builds = e->timed_builds;
    if (reset) {
      e->sum_s_ms = e->sum_h_ms = 0;
      e->sum_flops_h = e->sum_flops_s = e->timed_builds = 0;
    }
  });
}

int hsdla_b200_build_hs(const hsdla_b200_problem* p, const hsdla_b200_options* o, double* H, double* S,
                        hsdla_b200_stats* st) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    if (!p) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null problem"};
    check_dims(p->n_atoms, p->n_l, p->n_g);
    if (!H || !S) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null H or S"};
    if (!p->A || !p->B || !p->T_AA || !p->T_AB || !p->T_BB || !p->U)
      throw Fail{HSDLA_B200_DIMENSION_ERROR, "null problem pointer"};
    // streamed upload + build per GPU (chunk c+1's H2D overlaps chunk c's phases)
    one_shot(o, p->n_atoms, p->n_l, p->n_g, H, S, st, t0, [&](hsdla_b200_engine* e, uint64_t a0, int algo) {
      engine_build_streamed(e, p, a0, algo);
      return 0.0;
    });
  });
}

int hsdla_b200_build_hs_kpoints(const hsdla_b200_problem* common, uint64_t n_k, const uint64_t* n_g,
                                const double* const* A, const double* const* B, const hsdla_b200_options* o,
                                double* const* H, double* const* S, hsdla_b200_stats* st) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    if (!common) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null problem"};
    check_dims(common->n_atoms, common->n_l, common->n_g);
    if (!common->T_AA || !common->T_AB || !common->T_BB || !common->U)
      throw Fail{HSDLA_B200_DIMENSION_ERROR, "null operator / U pointer"};
    if (n_k == 0) return;
    if (!A || !B || !H || !S) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null k-point array"};
    uint64_t ng_max = 0;
    for (uint64_t k = 0; k < n_k; ++k) {
      if (!A[k] || !B[k] || !H[k] || !S[k]) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null k-point buffer"};
      const uint64_t ngk = n_g ? n_g[k] : common->n_g;
      check_dims(common->n_atoms, common->n_l, ngk);
      ng_max = std::max(ng_max, ngk);
    }
    if (o && o->n_gpus > 1) throw Fail{HSDLA_B200_CONFIG_ERROR, "k-point batches run on one GPU"};
    const int algo = o ? o->algo : HSDLA_B200_ALGO_REFINED_MERGED;
    if (!valid_algo(algo)) throw Fail{HSDLA_B200_CONFIG_ERROR, "unknown algo " + std::to_string(algo)};
    if (o && (o->flags & ~kKnownFlags)) throw Fail{HSDLA_B200_CONFIG_ERROR, "unknown option flags"};
    const std::vector<int> devs = devices_of(o);
    std::lock_guard<std::mutex> lk(g_cache_mu);
    const uint64_t ng0 = n_g ? n_g[0] : common->n_g;
    hsdla_b200_engine* e = get_engines(devs, common->n_atoms, common->n_l, ng0, 1, ng_max)->engines[0];
    HS_CUDA(cudaSetDevice(e->device));
    e->arith = o && (o->flags & HSDLA_B200_FLAG_ARITH_4M) ? HSDLA_B200_ARITH_4M : HSDLA_B200_ARITH_3M;
    engine_kpoints(e, common, n_k, n_g, A, B, algo, H, S);
    if (st) {
      engine_sync(e, st);  // the last k-point's device stats
      st->total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      flop_model(algo == HSDLA_B200_ALGO_ORIGINAL ? 0 : 1, common->n_atoms, common->n_l, e->ng, st->n_hpd,
                 st->ledger);
    } else {
      HS_CUDA(cudaStreamSynchronize(e->stream));
    }
  });
}

int hsdla_b200_problem_file_info(const char* path, uint64_t* n_atoms, uint64_t* n_l, uint64_t* n_g, uint8_t* hpd) {
  return guarded([&] {
    Fd f;
    f.fd = open_hsdl(path);
    const HsdlHeader h = read_hsdl_header(f.fd, path);
    if (n_atoms) *n_atoms = h.na;
    if (n_l) *n_l = h.nl;
    if (n_g) *n_g = h.ng;
    if (hpd) std::copy(h.hpd.begin(), h.hpd.end(), hpd);
  });
}

int hsdla_b200_engine_load(hsdla_b200_engine* e, const char* path, uint64_t atom_begin) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_load_file(e, path, atom_begin);
  });
}

int hsdla_b200_build_hs_file(const char* path, const hsdla_b200_options* o, double* H, double* S,
                             hsdla_b200_stats* st) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    HsdlHeader h;
    {
      Fd f;
      f.fd = open_hsdl(path);
      h = read_hsdl_header(f.fd, path);
    }
    check_dims(h.na, h.nl, h.ng);
    if (!H || !S) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null H or S"};
    // each GPU reads only its atom shard (and column window) from the file, then builds
    one_shot(o, h.na, h.nl, h.ng, H, S, st, t0, [&](hsdla_b200_engine* e, uint64_t a0, int algo) {
      const auto tl = std::chrono::steady_clock::now();
      engine_build_file(e, path, a0, algo);  // host file reads overlap the chunks' compute
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - tl).count();
    });
  });
}

}  // extern "C"
