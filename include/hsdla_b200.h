/* hsdla_b200 — B200-native (sm_100a) HSDLA Hamiltonian/Overlap construction.
 *
 * The C-ABI drop-in boundary for the reference's hot path
 *   hsdla::pipeline::build_hs_refined(const ProblemInstance&, const PipelineConfig&) -> HSResult
 *   (/root/reference/proj/include/hsdla/pipeline.hpp:55, src/pipeline.cpp:281-329)
 * Plain pointers and sizes only; no exceptions cross it.  Status codes map onto
 * the reference exception taxonomy (proj/include/hsdla/errors.hpp:9-26); the
 * message of the last failure on the calling thread is hsdla_b200_last_error().
 *
 * Storage contract (proj/include/hsdla/complex_matrix.hpp:11-31, problem.hpp:16-27):
 *   complex numbers are interleaved (re, im) doubles (std::complex<double>);
 *   A, B      : (n_atoms*n_l) x n_g, column-major, ld = n_atoms*n_l, atom blocks
 *               stacked rowwise (block a = rows [a*n_l, (a+1)*n_l));
 *   T_AA/T_AB/T_BB : n_atoms contiguous n_l x n_l column-major blocks; T_AA and
 *               T_BB are read from their LOWER triangles only (kernels.cpp:152-167);
 *               T^[BA] is never stored, it is T_AB^H (problem.hpp:15);
 *   U         : n_atoms*n_l reals (atom-major), S uses (U B)^H (U B) (pipeline.cpp:298-300);
 *   H, S      : n_g x n_g column-major; ONLY i >= j is written (lower triangle
 *               authoritative, complex_matrix.hpp:48-49), the strict upper
 *               triangle is never read or written, diagonal imaginary parts are
 *               exactly 0 (kernels.cpp:112,130,145).
 */
#ifndef HSDLA_B200_H
#define HSDLA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:9-26) ---------------------------------- */
#define HSDLA_B200_OK 0
#define HSDLA_B200_DIMENSION_ERROR 1 /* hsdla::DimensionError */
#define HSDLA_B200_SIZING_ERROR 2    /* hsdla::SizingError (incl. device out of memory) */
#define HSDLA_B200_CONFIG_ERROR 3    /* hsdla::ConfigError */
#define HSDLA_B200_IO_ERROR 4        /* hsdla::IoError */
#define HSDLA_B200_CUDA_ERROR 5      /* CUDA runtime / launch failure */
#define HSDLA_B200_NCCL_ERROR 6      /* NCCL failure */

/* ---- algorithms ------------------------------------------------------- */
/* Merged (default): Algorithm 3's sums restated per atom as H_a = Y_a^H M_a Y_a with
 * Y_a = [A_a; B_a] and the Hermitian block operator M_a = [[T_AA, T_AB], [T_AB^H, T_BB]]
 * (pipeline.cpp:302-324 evaluates the same sum as Z^H B + B^H Z + A^H (T_AA A)).  Phase
 * z_loop builds W_A = T_AA A + T_AB B and W_B = T_AB^H A + T_BB B (four per-atom
 * products); phase her2k is ONE lower-triangular contraction [A;B]^H [W_A;W_B] over 2K.
 * Executed 16 K N_G^2 + 32 N_A N_L^2 N_G complex-MAC flops against the ledger's
 * 20 K N_G^2 + 24 N_A N_L^2 N_G; hemm_loop and herkx report 0 s. */
#define HSDLA_B200_ALGO_REFINED_MERGED 0
/* Reference phase order s, z_loop, her2k, hemm_loop, herkx; five launches of the
 * contraction engine, executed flops == the reference ledger. */
#define HSDLA_B200_ALGO_REFINED 1
/* Same products as REFINED; her2k and herkx run as ONE lower-triangular contraction
 * over the stacked inner dimension [Z;B;A]^H [B;Z;X] (3K).  Executed flops == ledger;
 * the herkx phase reports 0 s (fused into her2k). */
#define HSDLA_B200_ALGO_REFINED_FUSED 3
/* The original algorithm (paper Algorithm 1, hsdla::pipeline::build_hs_original,
 * pipeline.cpp:189-279; Variant::Original): phases z_loop, her2k, s, chol_loop,
 * h_aa_update.  Per-atom Cholesky try/fail of T_AA on the GPU (bit-identical to
 * kernels::potrf), W_a = L_a^H A_a (trmm) for HPD atoms and T_AA A_a (hemm) for
 * the rest, then H += herk(B_T) + lower(A_f^H B_B) as ONE lower-triangular
 * contraction.  Ledger == flop_model(p, Original) with the observed n_hpd. */
#define HSDLA_B200_ALGO_ORIGINAL 2

/* ---- complex arithmetic of the contractions --------------------------------
 * 3M (default): Gauss's three-real-multiplication complex product, the ZGEMM3M
 *   scheme: per k, t1 += a_r b_r, t2 += a_i b_i, t3 += (a_r - a_i)(b_r + b_i), then
 *   Re = t1 + t2, Im = t3 - t1 + t2.  All FP64; 6 executed real flops per complex MAC
 *   (the ledger still counts 8), so a build is ~1/4 fewer tensor-core operations.
 *   Relative error stays at the 1e-15 level (the bar is 1e-11).
 * 4M: four real DMMAs per complex MAC, plain FP64 rounding per product. */
#define HSDLA_B200_ARITH_3M 0
#define HSDLA_B200_ARITH_4M 1
/* hsdla_b200_options.flags: force the 4M arithmetic for this call. */
#define HSDLA_B200_FLAG_ARITH_4M 1u
/* hsdla_b200_options.flags: multi-GPU calls sum H, S onto the first GPU (ncclReduce) and
 * download from it alone, instead of the default reduce-scatter where every GPU receives
 * and downloads its own slices of H and S. */
#define HSDLA_B200_FLAG_REDUCE_ROOT 2u

/* ---- the multi-GPU collective ------------------------------------------------
 * H and S are sums over atoms (pipeline.cpp:296-324): the GPUs of a column window hold
 * partial packed triangles of disjoint atom shards and sum them.  The result is reduced in
 * segments (the tile-column bands of the final H contraction when it runs banded, which
 * overlaps each band's reduce with the next band's compute; else the whole window).
 *   ROOT:    every segment summed onto rank `root` (ncclReduce).
 *   SCATTER: rank r of P owns the r-th of P equal slices of every segment (the last rank also
 *            the remainder): ncclReduceScatter in place, so each GPU receives 1/P of H and S
 *            and downloads its own slices over its own PCIe link (hsdla_b200_engine_owned). */
#define HSDLA_B200_REDUCE_ROOT 0
#define HSDLA_B200_REDUCE_SCATTER 1

/* Problem (ProblemInstance, problem.hpp:16-27). */
typedef struct hsdla_b200_problem {
  uint64_t n_atoms, n_l, n_g;
  const double* A;    /* 2 * n_atoms*n_l * n_g doubles */
  const double* B;    /* same */
  const double* T_AA; /* 2 * n_atoms * n_l*n_l doubles */
  const double* T_AB;
  const double* T_BB;
  const double* U;    /* n_atoms * n_l doubles */
} hsdla_b200_problem;

/* Options (PipelineConfig, pipeline.hpp:22-30, with the B200 strategy fields). */
typedef struct hsdla_b200_options {
  int n_gpus;             /* 0 or 1: one GPU; >1: a grid of col_groups column windows x
                             n_gpus / col_groups atom shards (see hsdla_b200_shard) */
  const int* device_ids;  /* NULL: devices 0..n_gpus-1.  A device may repeat: the engines that
                             share it are summed by a kernel instead of NCCL (single-GPU
                             emulation of the multi-GPU grid; every atom shard of a window must
                             then be on that one device) */
  int algo;               /* HSDLA_B200_ALGO_* */
  int flags;              /* HSDLA_B200_FLAG_ARITH_4M | HSDLA_B200_FLAG_REDUCE_ROOT */
  int col_groups;         /* 2-D tiling of H and S: number of column windows (must divide n_gpus).
                             0: automatic -- 1 (atom sharding only, H and S replicated per GPU)
                             unless the per-GPU memory estimate exceeds mem_budget_gb, then the
                             smallest divisor of n_gpus that fits */
  double mem_budget_gb;   /* per-GPU device memory for the automatic choice; 0: 90 % of free */
} hsdla_b200_options;

/* Phase slots = the reference's phase names (test_pipeline.cpp:167-176).  Refined
 * reports s, z_loop, her2k, hemm_loop, herkx; original reports z_loop, her2k, s,
 * chol_loop, h_aa_update (pipeline.cpp:207-276); unused slots are 0. */
#define HSDLA_B200_PHASE_S 0
#define HSDLA_B200_PHASE_Z_LOOP 1
#define HSDLA_B200_PHASE_HER2K 2
#define HSDLA_B200_PHASE_HEMM_LOOP 3
#define HSDLA_B200_PHASE_HERKX 4
#define HSDLA_B200_PHASE_CHOL_LOOP 5
#define HSDLA_B200_PHASE_H_AA_UPDATE 6
#define HSDLA_B200_N_PHASES 8

/* Ledger key order: gemm, hemm, her2k, herk, scaling, herkx, potrf, trmm, total
 * (flop_ledger.hpp; values == pipeline::flop_model, pipeline.cpp:336-364). */
typedef struct hsdla_b200_stats {
  double phase_seconds[HSDLA_B200_N_PHASES]; /* device time per phase slot, max over GPUs: from the
                                                 kernels' own %globaltimer stamps (first kernel's
                                                 start .. last kernel's end of each phase op) */
  double h2d_seconds;        /* host->device upload of A, B, T, U */
  double device_seconds;     /* first kernel's start .. last kernel's end (launch stamps); with a
                                multi-GPU reduce: CUDA events, first phase .. H,S reduced */
  double reduce_seconds;     /* NCCL reduce tail after the last contraction (0 on 1 GPU) */
  double d2h_seconds;        /* packed-triangle download + unpack into H, S */
  double total_seconds;      /* wall time of the call */
  uint64_t ledger[9];
  uint64_t executed_flops;   /* real flops the GPU executes (3M: 6 per complex MAC; ledger: 8) */
  uint64_t peak_device_bytes;/* device bytes held by the largest shard */
  uint64_t peak_temp_bytes;  /* device temporaries (the X/Z stacks), cf. HSResult::peak_temp_bytes */
  int n_gpus;
  int kernel_launches;       /* launches of this library's kernels in the build */
  uint64_t n_hpd;            /* atoms whose T_AA factorised (original algorithm; else n_atoms) */
  int col_groups;            /* column windows of the grid that ran (1: H, S replicated per GPU) */
  int reduce_mode;           /* HSDLA_B200_REDUCE_* of a multi-GPU call */
} hsdla_b200_stats;

/* ---- the drop-in --------------------------------------------------------
 * build_hs_refined (pipeline.cpp:281-329) on the GPU(s).  Writes the lower
 * triangles of the caller-allocated H and S (n_g*n_g complex each, col-major).
 * Engines (device buffers) are cached per (device, shape) across calls.  Host
 * buffers registered with hsdla_b200_host_register() are DMA'd directly; ordinary
 * pageable buffers are packed through pinned slabs by the host pool (streaming
 * stores, ~60 GB/s), both in atom chunks overlapped with the build. */
int hsdla_b200_build_hs(const hsdla_b200_problem* p, const hsdla_b200_options* opts, double* H,
                        double* S, hsdla_b200_stats* stats);

/* n_k k-points of one cell in one call (an extension beside the per-k-point drop-in): the
 * operators and U of `common` are k-independent and uploaded once; A[k], B[k] (same layout as
 * hsdla_b200_problem.A/B with n_g[k] columns; common->A/B unused) give each k-point's
 * coefficients and H[k], S[k] (n_g[k] x n_g[k]) receive its lower triangles.  n_g NULL: every
 * k-point has common->n_g G vectors; else the basis size may differ per k-point (N_G(k) of a
 * real FLAPW k-point set): the engine is allocated for the largest and re-targeted per k-point
 * without reallocation.  On one GPU (opts->n_gpus <= 1): while k-point k builds, k+1's
 * A, B are uploaded and k-1's H, S downloaded and unpacked, so the per-k-point cost approaches
 * the device-resident build.  Results equal n_k hsdla_b200_build_hs calls to FP64 rounding
 * (the per-call path chunks its uploads).  stats: the last k-point's, total_seconds = batch. */
int hsdla_b200_build_hs_kpoints(const hsdla_b200_problem* common, uint64_t n_k, const uint64_t* n_g,
                                const double* const* A, const double* const* B, const hsdla_b200_options* opts,
                                double* const* H, double* const* S, hsdla_b200_stats* stats);

/* ---- HSDL v1 problem files (problem.cpp:144-243) ---------------------------
 * Header of a file written by the reference's save_problem: dims and, when hpd
 * is non-NULL, n_atoms hpd flags.  Bad magic / version / truncation / missing
 * file -> HSDLA_B200_IO_ERROR (load_problem's IoError, test_io.cpp:47-63). */
int hsdla_b200_problem_file_info(const char* path, uint64_t* n_atoms, uint64_t* n_l, uint64_t* n_g, uint8_t* hpd);
/* build_hs(load_problem(path), cfg) without a host ProblemInstance: every GPU
 * streams only its atom shard (A/B rows of each column, T blocks, U) from the file
 * into HBM through pinned staging slabs, in atom chunks overlapped with the build.
 * Rows are copied out of a read-only mapping of the file that the engine keeps while
 * the file's (device, inode, size, mtime) are unchanged; the file must not be
 * truncated during a call.  Same outputs / stats contract as hsdla_b200_build_hs
 * (h2d_seconds = file load). */
int hsdla_b200_build_hs_file(const char* path, const hsdla_b200_options* opts, double* H, double* S,
                             hsdla_b200_stats* stats);

/* pipeline::flop_model (pipeline.cpp:336-364). variant: 0 original, 1 refined. */
int hsdla_b200_flop_model(int variant, uint64_t n_atoms, uint64_t n_l, uint64_t n_g, uint64_t n_hpd,
                          uint64_t ledger[9]);

/* kernels::potrf (kernels.cpp:417-436) for n_blocks lower-authoritative n_l x n_l
 * blocks (T, contiguous column-major blocks) on `device`.  L receives, per block,
 * the full factor (upper exactly 0) when it factorises, else the operand Q with
 * Q^H = T read from its lower triangle (full(T) with the diagonal conjugated: the
 * hemm operand the original algorithm falls back to);
 * pivot[b] = -1 on success, else the failing pivot (PotrfResult::pivot).  Same
 * operation order as the reference with no FMA contraction: bit-identical. */
int hsdla_b200_potrf(int device, uint64_t n_blocks, uint64_t n_l, const double* T, double* L, int64_t* pivot);

/* ---- the reference kernel layer on the GPU (hsdla::kernels, kernels.hpp:24-75) ---
 * Host matrices (interleaved complex, column-major, leading dimension in complex
 * elements); each call uploads, runs the sm_100a contraction engine and downloads.
 * alpha / beta marked `const double*` are complex (re, im).  Contracts of the
 * reference kernels: herk / her2k / herkx read and write only the LOWER triangle of
 * C (diagonal imaginary parts := 0, kernels.cpp:112,130,145); beta == 0 never
 * reads C; alpha == 0 only scales C by beta; hemm reads only H's lower triangle;
 * trmm uses only T's lower triangle.  ledger_flops (nullable) is INCREMENTED by the
 * reference's closed-form charge (kernels.cpp:254,296,316,339,363,390,444),
 * independent of alpha / beta.  Shapes as in kernels.hpp: herk A k x n; her2k /
 * herkx A, B k x n; gemm op(A) m x k, op(B) k x n (trans 0 None, 1 ConjTrans);
 * hemm H n x n, B, C n x m; trmm T n x n, B n x m in place; diag_scale X = diag(u) B
 * (X may alias B). */
int hsdla_b200_herk(int device, uint64_t n, uint64_t k, double alpha, const double* A, uint64_t lda, double beta,
                    double* C, uint64_t ldc, uint64_t* ledger_flops);
int hsdla_b200_her2k(int device, uint64_t n, uint64_t k, const double* alpha, const double* A, uint64_t lda,
                     const double* B, uint64_t ldb, double beta, double* C, uint64_t ldc, uint64_t* ledger_flops);
int hsdla_b200_herkx(int device, uint64_t n, uint64_t k, const double* alpha, const double* A, uint64_t lda,
                     const double* B, uint64_t ldb, double beta, double* C, uint64_t ldc, uint64_t* ledger_flops);
int hsdla_b200_gemm(int device, int trans_a, int trans_b, uint64_t m, uint64_t n, uint64_t k, const double* alpha,
                    const double* A, uint64_t lda, const double* B, uint64_t ldb, const double* beta, double* C,
                    uint64_t ldc, uint64_t* ledger_flops);
int hsdla_b200_hemm(int device, uint64_t n, uint64_t m, const double* alpha, const double* H, uint64_t ldh,
                    const double* B, uint64_t ldb, const double* beta, double* C, uint64_t ldc, uint64_t* ledger_flops);
int hsdla_b200_trmm(int device, int trans, uint64_t n, uint64_t m, const double* alpha, const double* T, uint64_t ldt,
                    double* B, uint64_t ldb, uint64_t* ledger_flops);
int hsdla_b200_diag_scale(int device, uint64_t rows, uint64_t cols, const double* u, const double* B, uint64_t ldb,
                          double* X, uint64_t ldx, uint64_t* ledger_flops);

/* generate_problem (problem.cpp:79-142), bit-identical to the reference
 * (std::mt19937_64 + the reference's double mapping).  Output layouts as above;
 * hpd: n_atoms bytes (hpd_flags). */
int hsdla_b200_generate_problem(uint64_t n_atoms, uint64_t n_l, uint64_t n_g, uint64_t seed,
                                uint64_t n_not_hpd, double* A, double* B, double* T_AA, double* T_AB,
                                double* T_BB, double* U, uint8_t* hpd);

/* generate_problem restricted to the atoms [atom_begin, atom_end) of the n_atoms-atom instance:
 * bit-identical to rows [atom_begin*n_l, atom_end*n_l) of A and B and blocks atom_begin..
 * atom_end-1 of T_AA, T_AB, T_BB, U, hpd of the full instance (the generator stream is skipped,
 * not stored), so each rank of a multi-GPU run generates only its own shard.  Output layouts
 * as above with n_atoms := atom_end - atom_begin (A, B leading dimension (atom_end-atom_begin)*n_l). */
int hsdla_b200_generate_problem_shard(uint64_t n_atoms, uint64_t n_l, uint64_t n_g, uint64_t seed,
                                      uint64_t n_not_hpd, uint64_t atom_begin, uint64_t atom_end, double* A,
                                      double* B, double* T_AA, double* T_AB, double* T_BB, double* U, uint8_t* hpd);

/* Contiguous, count-balanced atom ranges for `parts` GPUs:
 * bounds[r] .. bounds[r+1] is shard r; bounds has parts+1 entries. */
int hsdla_b200_shard_atoms(uint64_t n_atoms, int parts, uint64_t* bounds);
/* Row-balanced shards (what the multi-GPU drop-in uses): the K = n_atoms n_l rows split into
 * `parts` equal ranges; shard r is shards[4r .. 4r+3] = {atom_begin, n_atoms_local, row_begin,
 * row_end} (rows local to the shard, hsdla_b200_shard).  Shards' partials sum to the full H, S
 * (the sum over atoms of pipeline.cpp:296-324 regrouped by rows). */
int hsdla_b200_shard_rows(uint64_t n_atoms, uint64_t n_l, int parts, uint64_t* shards);

const char* hsdla_b200_last_error(void);
int hsdla_b200_device_count(int* count);
int hsdla_b200_host_register(void* ptr, size_t bytes);   /* cudaHostRegister (portable) */
int hsdla_b200_host_unregister(void* ptr);
int hsdla_b200_release_cache(void);                      /* free cached engines */

/* ---- device-resident engine (one per GPU / per rank) ---------------------
 * An engine owns the device copy of one atom shard [atom_begin, atom_end) of a
 * problem with n_atoms_total atoms, its temporaries and packed-lower partial
 * H and S.  build() runs the whole hot path on device-resident inputs (the
 * bench's `value`); download() returns the lower triangles. */
typedef struct hsdla_b200_engine hsdla_b200_engine;

int hsdla_b200_engine_create(int device, uint64_t n_atoms_local, uint64_t n_l, uint64_t n_g,
                             hsdla_b200_engine** out);
/* An engine for one shard of a multi-GPU grid: n_atoms_local atoms (an atom shard; the reduce
 * sums the shards' partials) and the COLUMN WINDOW [col_begin, col_end) of H and S (2-D
 * owner-computes tiling for N_G too large to replicate H and S on every GPU: engines of
 * different windows compute disjoint tile-column bands of the lower triangle, no exchange).
 * A window holds the operand columns [col_begin, n_g) (its tiles' rows) and the packed range
 * of its columns.  col_end 0 means n_g; col_begin and col_end (unless n_g) are multiples of 64.
 * n_g_capacity >= n_g (0: n_g) sizes a whole-window engine for later hsdla_b200_engine_reshape
 * to other N_G without reallocation. */
typedef struct hsdla_b200_shard {
  uint64_t n_atoms_local, n_l, n_g;
  uint64_t col_begin, col_end;
  uint64_t n_g_capacity;
  /* K-row range [row_begin, row_end) of the shard's n_atoms_local * n_l rows that its H/S
   * contractions sum over (row_end 0: all rows).  A row-balanced grid (hsdla_b200_shard_rows)
   * gives every GPU the same share of the contraction work; the range must start in the
   * shard's first atom and end in its last (boundary atoms are held by two shards). */
  uint64_t row_begin, row_end;
} hsdla_b200_shard;
int hsdla_b200_engine_create_shard(int device, const hsdla_b200_shard* shard, hsdla_b200_engine** out);
/* Re-target the engine at N_G = n_g (whole window) within its capacity; HSDLA_B200_SIZING_ERROR
 * if it does not fit.  Inputs must be uploaded again. */
int hsdla_b200_engine_reshape(hsdla_b200_engine* e, uint64_t n_g);
int hsdla_b200_engine_destroy(hsdla_b200_engine* e);
/* H2D of atoms [atom_begin, atom_begin + n_atoms_local) of p (p->n_atoms total). */
int hsdla_b200_engine_upload(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t atom_begin);
/* Stream atoms [atom_begin, atom_begin + n_atoms_local) of an HSDL v1 file into
 * the engine (pinned double-buffered pread -> H2D on the copy stream). */
int hsdla_b200_engine_load(hsdla_b200_engine* e, const char* path, uint64_t atom_begin);
/* Device-side synthetic inputs for timing sweeps (A, B, T ~ U(-1,1), U ~ U(0.5,1.5),
 * counter-based hash of `seed`; NOT the reference generator). */
int hsdla_b200_engine_fill_synthetic(hsdla_b200_engine* e, uint64_t seed);
/* Complex arithmetic of this engine's contractions (HSDLA_B200_ARITH_*); new engines
 * and the kernel layer take the process default, set by hsdla_b200_set_default_arith. */
int hsdla_b200_engine_set_arith(hsdla_b200_engine* e, int arith);
int hsdla_b200_set_default_arith(int arith);
/* on != 0: this engine's builds run their final H contraction in tile-column bands, so an
 * hsdla_b200_engine_download enqueued right after the build overlaps H's D2H and host
 * unpack with the remaining bands (as the one-shot drop-in does); S's download already
 * overlaps the H phases.  Costs ~1 % of device time (smaller final launches); off by
 * default (device-resident builds that are not downloaded). */
int hsdla_b200_engine_set_download_overlap(hsdla_b200_engine* e, int on);
/* Enqueue the full build (all phases) on the engine stream; asynchronous. */
int hsdla_b200_engine_build(hsdla_b200_engine* e, int algo);
/* Streamed build from HOST memory: uploads shard `atom_begin` of p in atom chunks on
 * a copy stream, each chunk's phases start as soon as its bytes land, H and S
 * accumulate over chunks.  Asynchronous w.r.t. the host for pinned p; follow with
 * reduce / sync / download as for engine_build. */
int hsdla_b200_engine_build_streamed(hsdla_b200_engine* e, const hsdla_b200_problem* p, uint64_t atom_begin,
                                     int algo);
/* NCCL sum of the packed partial H and S over the engine's communicator (no-op without one),
 * in the engine's reduce mode (HSDLA_B200_REDUCE_ROOT onto rank `root`, the default, or
 * HSDLA_B200_REDUCE_SCATTER).  Every rank of the communicator calls it. */
int hsdla_b200_engine_reduce(hsdla_b200_engine* e, int root);
int hsdla_b200_engine_set_reduce_mode(hsdla_b200_engine* e, int mode);
/* The reduce of a group of engines of THIS process that share a column window (disjoint atom
 * shards): with communicators (one per engine, one rank each, e.g. from ncclCommInitAll) the
 * NCCL calls of all engines are grouped; engines without one must share a device and are
 * summed by a deterministic kernel (rank order).  engines[r] is rank r. */
int hsdla_b200_group_reduce(hsdla_b200_engine* const* engines, int n, int mode, int root);
/* The packed-lower index ranges (global, [begin, end) pairs) of H and S this engine holds final
 * values for after the last build / reduce -- what hsdla_b200_engine_download writes.  ranges
 * holds 2 * max entries; *n receives the count (which may exceed max). */
int hsdla_b200_engine_owned(hsdla_b200_engine* e, uint64_t* ranges, uint64_t max, uint64_t* n);
/* Wait for the engine's streams; fills phase/device timings of the last build. */
int hsdla_b200_engine_sync(hsdla_b200_engine* e, hsdla_b200_stats* stats);
/* D2H of the packed ranges this engine owns (all of its window before a reduce; its slices
 * after a SCATTER reduce; everything on the root / nothing elsewhere after a ROOT reduce),
 * unpacked into the lower triangles of the n_g x n_g matrices H, S (either may be NULL).
 * Synchronous. */
int hsdla_b200_engine_download(hsdla_b200_engine* e, double* H, double* S);
/* Packed lower (LAPACK 'L' packed, column-major) device pointers of H and S. */
int hsdla_b200_engine_device_results(hsdla_b200_engine* e, void** Hp, void** Sp);
/* The cudaStream_t the engine launches on. */
int hsdla_b200_engine_stream(hsdla_b200_engine* e, void** stream);
/* NCCL: one communicator per engine (one rank per GPU; id from rank 0).  id128 NULL
 * with nranks 1 drops the communicator (reduce becomes a no-op); an id with nranks 1
 * builds a single-rank communicator, so the reduce path runs through NCCL. */
int hsdla_b200_nccl_unique_id(void* id128);
int hsdla_b200_engine_set_comm(hsdla_b200_engine* e, const void* id128, int nranks, int rank);

/* Contraction-kernel timing for the roofline: mean CUDA-event duration (ms) of
 * the S contraction (herk+herk, 8 K N_G^2 flops) and the H contraction launch
 * (fused: 12 K N_G^2; merged: 8 K N_G^2; refined algo: the her2k launch, 8 K N_G^2) over every
 * build since the last reset, recorded on the engine stream without per-build
 * host syncs.  reset != 0 clears the accumulators after reading. */
int hsdla_b200_engine_kernel_times(hsdla_b200_engine* e, int reset, double* ms_s, double* ms_h,
                                   uint64_t* flops_s, uint64_t* flops_h, uint64_t* n_builds);

/* Roofline denominator: runs a DMMA (mma.sync m8n8k4 f64) throughput loop on
 * `device` for about `seconds` and returns the achieved FP64 TFLOP/s.  A
 * measurement probe, not part of the H/S path. */
int hsdla_b200_fp64_peak(int device, double seconds, double* tflops);

/* ---- LAPW matching-coefficient setup (north_star subsystem 1) -------------
 * Builds A, B and U on the GPU from the physical inputs instead of uploading
 * them.  The reference has no implementation of this step (A, B
 * are synthetic inputs there); the math is the standard LAPW matching of paper
 * Eq. (basis), see paper_1712_07206_b200/csrc/lapw_setup.cuh:
 *   A^{a,G}_lm = c [j_l(KR) udot'_l - K j_l'(KR) udot_l] / det,
 *   B^{a,G}_lm = c [K j_l'(KR) u_l - j_l(KR) u'_l] / det,
 *   c = 4 pi Omega^{-1/2} e^{iK.tau_a} i^l conj(Y_lm(K^)),  K = k + G,
 *   det = u_l udot'_l - udot_l u'_l   (radial values at R = rmt of the atom's type),
 * rows a*(lmax+1)^2 + l(l+1)+m, Y_lm with the Condon-Shortley phase; U row
 * a*(lmax+1)^2 + lm = udot_norm[type(a)][l]. */
typedef struct hsdla_b200_lapw {
  uint64_t n_atoms, n_types, n_g;
  int lmax;                  /* <= 20; N_L = (lmax+1)^2 */
  double kpt[3];             /* k-point, Cartesian */
  double omega;              /* unit-cell volume */
  const double* gvec;        /* n_g x 3 Cartesian G vectors (G_j = gvec[3j..3j+2]) */
  const double* tau;         /* n_atoms x 3 Cartesian atom positions */
  const int32_t* atom_type;  /* n_atoms, in [0, n_types) */
  const double* rmt;         /* n_types muffin-tin radii */
  const double* u;           /* n_types x (lmax+1), row-major: u_l(R) */
  const double* du;          /* u_l'(R) */
  const double* udot;        /* udot_l(R) */
  const double* dudot;       /* udot_l'(R) */
  const double* udot_norm;   /* ||udot_l|| (the U diagonal) */
} hsdla_b200_lapw;

/* One-shot: A, B ((n_atoms (lmax+1)^2) x n_g complex, col-major) and U to host. */
int hsdla_b200_lapw_coefficients(int device, const hsdla_b200_lapw* sys, double* A, double* B, double* U);
/* Fill the engine's A, B, U for its shard [atom_begin, atom_begin + n_atoms_local) in HBM. */
int hsdla_b200_engine_setup_lapw(hsdla_b200_engine* e, const hsdla_b200_lapw* sys, uint64_t atom_begin);
/* H2D of the shard's T_AA, T_AB, T_BB blocks only (with setup_lapw: a build needs no A/B upload).
 * Asynchronous, on the engine's copy stream (after the previous build is done with T); the next
 * build's S contraction runs meanwhile and its operator expansion waits for the copies.  Page-
 * locked sources must stay valid until that build has been synchronised. */
int hsdla_b200_engine_upload_operators(hsdla_b200_engine* e, const double* T_AA, const double* T_AB,
                                       const double* T_BB, uint64_t atom_begin);
/* CUDA-event times (ms) of the last setup_lapw: both kernels (ms) and the HBM-write
 * stream kernel alone (ms_stream, nullable), and the bytes written. */
int hsdla_b200_engine_setup_time(hsdla_b200_engine* e, double* ms, uint64_t* bytes, double* ms_stream);

#ifdef __cplusplus
}
#endif
#endif /* HSDLA_B200_H */
