// The per-GPU device engine of the HSDLA refined H/S construction (drop-in for
// hsdla::pipeline::build_hs_refined, reference pipeline.cpp:281-329).
//
// Device data layout (one engine per GPU / shard, all HBM-resident):
//   A, B    K x ncol complex, column-major, ld = K (the reference stacking,
//           problem.hpp:20-21), columns [c0, N_G) of the problem; two sets when a
//           k-point batch alternates them (set 1 allocated on first use)
//   X1      K x ncol: first U*B (phase s, diag_scale kernels.cpp:438-450), then W_A
//           (merged) or T_AA A (hemm_loop, pipeline.cpp:314-321)
//   X2      K x ncol: W_B (merged) or Z = T_AB^H A + 1/2 T_BB B (z_loop, pipeline.cpp:302-307)
//   Tab     raw per-atom T_AB blocks (used as-is: Z = T_AB^H A is a CTN product)
//   Pbb,Paa 1/2 full(T_BB) (full(T_BB) for the merged algorithm), full(T_AA) expanded
//           from the LOWER triangles only
//   Wl      merged algorithm: the left operand of W = M Y per atom, 4 N_L^2 complex:
//           [Paa | Tab] (N_L k over A_a's rows x 2 N_L output rows), then [Pab | Pbb]
//           (k over B_a's rows) with Pab = T_AB^H, Pbb = full(T_BB); one BATCH launch
//           writes W_A (rows < N_L) to X1 and W_B to X2
//   Hp, Sp  the engine's column window [c0, c1) of packed-lower N_G x N_G storage:
//           global packed indices [pk0, pk0 + npk) (LAPACK 'L' packing; halves D2H and
//           NCCL bytes).  The whole triangle when the window is [0, N_G).
//
// Shards.  An engine holds n_atoms_local atoms of a problem (the atom shard: its
// partial H, S are summed over shards by the reduce) and one COLUMN WINDOW of H and S
// (2-D owner-computes tiling for N_G too large to replicate H and S: engines of
// different windows compute disjoint tile-column bands of the lower triangle and
// never exchange data).  A window [c0, c1) needs the operand columns [c0, N_G) (the
// rows i >= j of its tiles), so its A, B, X hold ncol = N_G - c0 columns.
//
// The merged algorithm (default) restates Algorithm 3 as one contraction per matrix:
// per atom, H_a = Y_a^H M_a Y_a with Y_a = [A_a; B_a] and the Hermitian block operator
// M_a = [[T_AA, T_AB], [T_AB^H, T_BB]] (the same sum pipeline.cpp:302-324 evaluates as
// Z^H B + B^H Z + A^H (T_AA A)), so H = [A; B]^H [W_A; W_B] with W_A = T_AA A + T_AB B in
// X1 and W_B = T_AB^H A + T_BB B in X2: 16 K N_G^2 contraction flops instead of 20.
//
// A build is a list of atom CHUNKS.  The device-resident build is one chunk over
// all atoms.  The streamed build (the one-shot drop-in with host buffers) splits
// the atoms into chunks: chunk c+1 is copied host->device on the copy stream while
// chunk c's phases run, and every contraction accumulates into H, S (beta = 1 after
// the first chunk) — H and S are sums over atoms, so any chunking is exact up to
// FP64 rounding order.  S is downloaded and unpacked on the host while H computes.
// A k-point batch (hsdla_b200_build_hs_kpoints) alternates the two A/B sets so the next
// k-point's upload and the previous one's download overlap the current build.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <sys/stat.h>

#include <chrono>
#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"
#include "ctn_params.hpp"

namespace hsdla_b200 {

// One atom chunk [a0, a1) of a build over one A/B set: the parameter blocks of every launch.
struct ChunkPlan {
  uint64_t a0 = 0, a1 = 0;
  const double2* A = nullptr;  // the set's A / B (raw-pointer launches: diag_scale, select_left)
  const double2* B = nullptr;
  // s: S; z: Z -> X1 (refined/original); zf: Z -> X2 (fused); x: Q^H A -> X1;
  // h: fused her2k+herkx; h2k: her2k over X1; hkx: herkx A^H X1; haa: original X2^H X1
  // merged: w: [W_A; W_B] = M Y (W_A = T_AA A + T_AB B -> X1, W_B = T_AB^H A + T_BB B -> X2,
  // one launch); hm: [A;B]^H [X1;X2]
  CtnParams s, z, zf, x, h, h2k, hkx, haa, w, hm;
  // the S contraction split by segment (first streamed chunk: A^H A starts on A's rows
  // while B, T, U are still on the wire; (UB)^H (UB) accumulates once they landed)
  CtnParams sA, sB;
  dim3 grid_tri, grid_bat, grid_batw;
  int w_bn = 0;  // the W launch's tile width (kBatWBN or kBatBN)
};

struct OpTime {
  int phase;
  int s0, s1;  // the launch timestamp slots [s0, s1) of its kernels (stamp.cuh)
};

// A packed-lower index range [b0, b1) (global indices) of S (h == 0) or H (h == 1) copied to
// the host stage at local offset b0 - pk0 (+ cap_pk for S) and final once `ready` (on the
// copy stream) has completed.
struct DlPiece {
  int h;
  uint64_t b0, b1;
  cudaEvent_t ready;
};
// The download of one build, snapshotted at enqueue time (the engine may be reshaped
// for the next k-point before the host unpacks this one); pieces in landing order.
struct Download {
  uint64_t ng = 0, pk0 = 0;
  std::vector<DlPiece> seq;
  bool pending = false;
};

// Collective mode of hsdla_b200_engine_reduce (include/hsdla_b200.h HSDLA_B200_REDUCE_*).
enum ReduceMode { kReduceRoot = 0, kReduceScatter = 1 };

}  // namespace hsdla_b200

struct hsdla_b200_engine {
  int device = 0;
  // ---- geometry ----
  uint64_t na = 0, nl = 0, K = 0;  // local atoms, K = na * nl
  // K-row range [row0, row1) of the local stack that this engine's H/S contractions sum over
  // (default [0, K)).  A row-balanced multi-GPU grid splits the global K rows evenly, so an
  // engine holds every atom its rows touch (boundary atoms on two engines: their W / Z / X
  // are computed on both, their rows contracted on one).  Atoms [own_a0, own_a1) are the ones
  // whose first row is in range (each atom of the grid is owned once: the n_hpd count).
  uint64_t row0 = 0, row1 = 0, own_a0 = 0, own_a1 = 0;
  uint64_t ng = 0;                 // N_G of the problem (global)
  uint64_t c0 = 0, c1 = 0;         // H/S column window [c0, c1)
  uint64_t ncol = 0;               // operand columns held: [c0, ng)
  uint64_t pk0 = 0, npk = 0;       // window's global packed range [pk0, pk0 + npk)
  uint64_t cap_cols = 0, cap_pk = 0;  // allocated capacity (columns of A/B/X, packed elements)
  // ---- streams / buffers ----
  cudaStream_t stream = nullptr, copy_stream = nullptr, comm_stream = nullptr;
  double2* Aset[2] = {};  // A/B sets (set 1: k-point batches)
  double2* Bset[2] = {};
  double2 *X1 = nullptr, *X2 = nullptr;
  double2 *Tab = nullptr, *Taa = nullptr, *Tbb = nullptr, *Paa = nullptr, *Pbb = nullptr, *Wl = nullptr;
  double* U = nullptr;
  int32_t* info = nullptr;        // per-atom potrf result of the original algorithm (-1 = HPD)
  int* n_fail = nullptr;          // original algorithm: failed atoms so far in this build
  double2 *Hp = nullptr, *Sp = nullptr;
  double2* host_stage = nullptr;  // pinned, 2 * cap_pk (H at [0, npk), S at [cap_pk, cap_pk + npk))
  double2* host_stage_x[2] = {};  // download slots 1, 2 (k-point batches), same layout
  int sms = 148;                  // persistent TRI grid
  double* sk_ws = nullptr;        // stream-K workspace (sms slots x 64x64 complex)
  uint32_t* sk_flags = nullptr;
  uint32_t epoch = 0;
  uint64_t device_bytes = 0, temp_bytes = 0;
  // ---- collective group (ranks that share this window; their partials are summed) ----
  ncclComm_t comm = nullptr;
  bool comm_owned = true;         // false: the communicator belongs to the drop-in's cache
  std::vector<hsdla_b200_engine*> local_group;  // same-device group reduced by a sum kernel (no NCCL)
  int nranks = 1, rank = 0;
  int red_mode = hsdla_b200::kReduceRoot;
  int red_root = 0;

  std::vector<hsdla_b200::ChunkPlan> whole, streamed, streamed_pg;  // streamed: pinned / pageable feed
  bool streamed_dirty = true;                                       // streamed plans need a rebuild
  std::vector<hsdla_b200::ChunkPlan> whole2;                        // set 1 (k-point batches)
  cudaStream_t h2d_stream = nullptr;
  cudaEvent_t ev_kup[2] = {}, ev_kbuilt[2] = {};
  cudaEvent_t wait_before_s = nullptr, wait_before_h = nullptr;  // next enqueue_chunk waits (storage reuse)
  // per-build timing
  // launch timestamp slots of the current build (stamp.cuh): every kernel of a timed phase stamps
  // one; engine_sync reads them back for the phase times and the device time
  static constexpr int kMaxStamps = 1024;
  unsigned long long* d_stamp = nullptr;
  int stamp_used = 0;
  std::vector<hsdla_b200::OpTime> ops;
  // ev_end: the build's end (ordering only).  ev_begin / ev_end_t: timing events around the build,
  // recorded only by engines that reduce with others (their reduce is timed by events)
  bool marks_timed = false;  // this build recorded ev_begin / ev_end_t (grouped when it began)
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr, ev_end_t = nullptr, ev_s_done = nullptr, ev_s_red = nullptr,
              ev_reduce_end = nullptr, ev_up0 = nullptr, ev_up1 = nullptr,
              ev_a0 = nullptr,   // the first streamed chunk's A rows landed
              ev_ops = nullptr,  // operators uploaded on the copy stream (engine_upload_operators)
              ev_cs_order = nullptr;  // copy_after_compute
  bool ops_pending = false;      // the next build must wait for ev_ops before expanding T
  static constexpr int kD2hPieces = 8;   // H downloads in column-range pieces, unpacked as each lands
  cudaEvent_t ev_h_band[kD2hPieces] = {};  // final H contraction finished tile-column band q
  cudaEvent_t ev_h_red[kD2hPieces] = {};   // ... and band q's packed range is reduced
  int piece_tiles[kD2hPieces + 1] = {};    // tile-column boundaries of the pieces / bands
  bool band_final_h = false;               // this build runs its final H contraction band by band
  bool overlap_dl = false;                 // engine builds band their final H (a download follows)
  bool banded = false;                     // ... and the last build did
  // download pieces: events recorded on the copy stream (S: up to 1, H: up to kD2hPieces).
  // Slot 0 serves every build; a k-point batch rotates over 2 or 3 slots (stage, events,
  // record) so k's D2H is enqueued before the host unpacks an earlier k-point.
  static constexpr int kDlSlots = 3;
  cudaEvent_t ev_dl_s = nullptr;
  cudaEvent_t ev_dl_h[kD2hPieces] = {};
  hsdla_b200::Download dl;                 // the enqueued, not yet unpacked download
  cudaEvent_t ev_dlx_s[2] = {};            // slots 1, 2 (created with host_stage_x)
  cudaEvent_t ev_dlx_h[2][kD2hPieces] = {};
  hsdla_b200::Download dlx[2];
  std::vector<cudaEvent_t> ev_chunk_up;
  int last_algo = 0, launches = 0;
  int arith = HSDLA_B200_ARITH_3M;  // complex product scheme of the contractions
  uint64_t n_hpd_last = 0;
  bool built = false, reduced = false, uploaded_streamed = false;
  cudaEvent_t ev_setup0 = nullptr, ev_setup1 = nullptr;  // last LAPW setup (tables + stream kernels)
  cudaEvent_t ev_setup_mid = nullptr;                      // between the two kernels
  uint64_t setup_bytes = 0;
  void* lapw_scratch = nullptr;  // device copy of the LAPW inputs (grown on demand)
  size_t lapw_scratch_bytes = 0;
  // pinned staging slabs for pageable inputs and HSDL files, allocated on first use
  static constexpr int kStageSlabs = 4;  // used round robin (8 measured no better)
  char* stage_buf[kStageSlabs] = {};
  cudaEvent_t stage_ev[kStageSlabs] = {};
  bool stage_busy[kStageSlabs] = {};
  int stage_next = 0;
  // HSDL file view: a read-only mapping of the last file this engine loaded, kept while the
  // file's (device, inode, size, mtime) stay the same, so repeated k-point calls on one file
  // copy rows straight out of the page cache without a pread per column piece
  const char* fmap = nullptr;
  size_t fmap_len = 0;
  struct stat fmap_st {};
  double tr_pack_ms = 0, tr_wait_ms = 0;  // HSDLA_B200_TRACE: pageable staging accounting
  // HSDLA_B200_TRACE: device timeline marks (timing events on the compute / copy streams),
  // printed relative to the first mark by finish_download
  std::vector<std::pair<std::string, cudaEvent_t>> tr_marks;
  std::vector<cudaEvent_t> tr_pool;
  uint64_t tr_pack_bytes = 0;
  // roofline: events around the whole-build S and H contraction launches, harvested lazily
  static constexpr int kRing = 64;
  struct KTimer {
    cudaEvent_t s0 = nullptr, s1 = nullptr, h0 = nullptr, h1 = nullptr;
    bool pending = false;
    uint64_t flops_h = 0, flops_s = 0;
  } ring[kRing];
  uint64_t builds = 0;
  double sum_s_ms = 0, sum_h_ms = 0;
  uint64_t sum_flops_h = 0, sum_flops_s = 0, timed_builds = 0;

  double2* A(int set = 0) const { return Aset[set]; }
  double2* B(int set = 0) const { return Bset[set]; }
};

namespace hsdla_b200 {

// Engine shard description (hsdla_b200_shard in the C-ABI, with defaults resolved).
struct ShardSpec {
  uint64_t na = 0, nl = 0, ng = 0;
  uint64_t row0 = 0, row1 = 0;   // contracted local K rows; row1 == 0: [0, na * nl)
  uint64_t c0 = 0, c1 = 0;       // column window; c1 == 0: [0, ng)
  uint64_t ng_capacity = 0;      // allocate for up to this N_G (0: ng)
};

constexpr size_t kStageSlab = size_t(64) << 20;

void check_dims(uint64_t na, uint64_t nl, uint64_t ng);
bool valid_algo(int algo);
hsdla_b200_engine* engine_create(int device, const ShardSpec& spec);
void engine_free(hsdla_b200_engine* e);
// Re-target an engine at N_G = ng (column window [c0, c1), c1 == 0: whole) within its
// allocated capacity; false (engine unchanged) if it does not fit.  Waits for the engine.
bool engine_reshape(hsdla_b200_engine* e, uint64_t ng, uint64_t c0 = 0, uint64_t c1 = 0);
void engine_upload(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0);
void engine_fill_synthetic(hsdla_b200_engine* e, uint64_t seed);
void engine_build(hsdla_b200_engine* e, int algo);
void engine_build_streamed(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t a0, int algo);
void engine_kpoints(hsdla_b200_engine* e, const hsdla_b200_problem* common, uint64_t nk, const uint64_t* ngk,
                    const double* const* A, const double* const* B, int algo, double* const* H, double* const* S);
void engine_reduce(hsdla_b200_engine* e, int root);
// The sum of the partials of a group of engines (same window, disjoint atom shards): NCCL
// (every engine has a communicator; grouped calls across the engines of this process) or,
// for engines that share one device, a deterministic sum kernel.  mode kReduceRoot: the
// whole result on rank `root`; kReduceScatter: every rank owns a contiguous slice of each
// band (hsdla_b200_engine_owned).  Overlaps the H phases band by band.
void group_reduce(const std::vector<hsdla_b200_engine*>& g, int mode, int root);
void engine_sync(hsdla_b200_engine* e, hsdla_b200_stats* st);
// Enqueue the D2H of the packed ranges this engine owns (all of them before a reduce),
// then unpack them into the lower triangles of H, S (either may be null).
// slot 1, 2: the further stages / event sets of k-point batches.
void enqueue_download(hsdla_b200_engine* e, int slot = 0);
void finish_download(hsdla_b200_engine* e, double* H, double* S,
                     std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), int slot = 0);
// The last event of a slot's download (the next build reusing H / S storage waits on it).
cudaEvent_t download_done_s(hsdla_b200_engine* e, int slot);
cudaEvent_t download_done_h(hsdla_b200_engine* e, int slot);
void engine_download(hsdla_b200_engine* e, double* H, double* S);
// Packed ranges of the current result this engine holds final values for.
std::vector<std::pair<uint64_t, uint64_t>> engine_owned(const hsdla_b200_engine* e);
uint64_t executed_flops(uint64_t na, uint64_t nl, uint64_t ng, int arith, int algo, uint64_t rows = 0);
void flop_model(int variant, uint64_t na, uint64_t nl, uint64_t ng, uint64_t n_hpd, uint64_t* l);
float ev_ms(cudaEvent_t a, cudaEvent_t b);
void harvest(hsdla_b200_engine* e, hsdla_b200_engine::KTimer& t);

// building blocks shared with the HSDL-file and LAPW front ends
void begin_build(hsdla_b200_engine* e, int algo);
void ensure_streamed_plans(hsdla_b200_engine* e);
void trace_mark(hsdla_b200_engine* e, cudaStream_t s, const std::string& what);
// The copy stream waits for everything enqueued on the compute stream so far (the previous
// build, and uploads engine_upload issued there) before it overwrites the inputs.
void copy_after_compute(hsdla_b200_engine* e);
// The build's begin / end marks on the compute stream (ev_end: ordering; timing events only
// for engines that reduce with others).
void mark_build_begin(hsdla_b200_engine* e);
void mark_build_end(hsdla_b200_engine* e);
void enqueue_chunk(hsdla_b200_engine* e, ChunkPlan& cp, int algo, bool last, hsdla_b200_engine::KTimer* kt,
                   bool s_rest = false);
// Row pitch of a packed staging slab: each column's rows start on a 4 KB boundary.  A 2-D H2D
// from rows packed back to back crosses host pages mid-row and runs at 22 / 40 GB/s for 2.6 /
// 6.5 KB rows; 4 KB-aligned rows go at 53-55 (the link rate; tools/h2d_rows.cu).
inline size_t slab_pitch(size_t colb) { return (colb + 4095) & ~size_t(4095); }
char* stage_acquire(hsdla_b200_engine* e, int& slot);
void stage_release(hsdla_b200_engine* e, int slot, cudaStream_t s);

// HSDL v1 files (hsdl_file.cpp)
void engine_load_file(hsdla_b200_engine* e, const char* path, uint64_t a0);
void engine_build_file(hsdla_b200_engine* e, const char* path, uint64_t a0, int algo);
void release_file_view(hsdla_b200_engine* e);

}  // namespace hsdla_b200
