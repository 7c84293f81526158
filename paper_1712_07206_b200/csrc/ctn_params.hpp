// Parameter block of the contraction engine (ctn_contract.cuh), visible to host code.
#pragma once

#include <cuda.h>
#include <vector_types.h>

#include <cstdint>

namespace hsdla_b200 {

constexpr int kMaxSeg = 3;
constexpr int kChunkC = 8;  // complex k per TMA slab (128 B rows)
constexpr int kStampWords = 4;  // words per launch timestamp slot (stamp.cuh)

// kTri: the strictly-lower tiles of the triangle (or of a column window); kTriDiag: its diagonal
// tiles (a launch of their own with a warp remapping, ctn_contract.cuh); kBatch: per-atom products.
// kTriRow: the last tile row when N_G leaves it ragged (a launch of its own, ctn_contract.cuh).
enum CtnMode { kTri = 0, kBatch = 1, kTriDiag = 2, kTriRow = 3 };

struct alignas(64) CtnParams {
  CUtensorMap L[kMaxSeg];  // left operands (conjugated), 3-D maps
  CUtensorMap R[kMaxSeg];  // right operands
  int kchunks[kMaxSeg];    // 8-complex slabs per segment
  int l_row_z[kMaxSeg];    // 1: tile row coordinate in dim 2, atom in dim 1; 0: row in dim 1, atom in dim 2
  int r_row_z[kMaxSeg];
  int half_last[kMaxSeg];  // BATCH: the segment's last 8-complex slab has <= 4 valid k (its
                           // second half is zero-fill and is skipped); 0 elsewhere
  int nseg;
  int n;                   // TRI: order N_G.  BATCH: number of output columns (N_G)
  int m_valid;             // BATCH: valid output rows per atom (N_L; 2 N_L for the stacked W = M Y)
  int m_row;               // BATCH, optional: rows per atom of `out` (0: m_valid).  Output rows
                           // i >= m_row go to out2 (row i - m_row): the stacked W_A / W_B split
  int tiles;               // TRI: tiles per dimension
  int tiles_total;         // TRI: lower tiles t(t+1)/2
  int band;                // TRI: tile-row band of the grouped tile order (>= 1)
  int col_t0, col_t1;      // TRI, optional: only the lower tiles with col_t0 <= tj < col_t1
                           // (col_t1 == 0: the whole lower triangle); tiles_total = their count
  int diag_t0;             // TRI diagonal launch: tile index of its first diagonal tile;
                           // ragged-row launch: tile column of its first tile
  int row_ti, row_v;       // ragged-row launch: the row's tile index, its valid 8-row fragment rows
  int with_diag;           // TRI: 1 = this launch covers the diagonal tiles too (small triangles:
                           // one launch; no warp remapping), 0 = strictly-lower tiles only
  int g0;                  // TRI: global column of the operands' first held column (a column
                           // window's engine holds columns [g0, n)); TMA coordinate = global - g0
  uint64_t pk0;            // TRI: global packed index of out[0] (the window's first packed element)
  double2* out;            // TRI: packed lower.  BATCH: column-major stacked buffer
  double2* out2;           // BATCH, optional: second stacked buffer (rows i >= m_row)
  double* sk_ws;           // TRI stream-K: per-CTA partial-accumulator slots
  uint32_t* sk_flags;      // TRI stream-K: per-CTA publish flags (== epoch when the slot is ready)
  uint32_t epoch;          // TRI stream-K: unique per launch
  uint64_t ldo;            // BATCH: output leading dimension (complex elements)
  int bat_tx, bat_ty;      // BATCH: column tiles, row tiles per atom
  int bat_tiles;           // BATCH: bat_tx * bat_ty * atoms (persistent CTAs loop over them)
  const int* keep_diag_imag;  // TRI, optional: when non-null and *keep_diag_imag != 0 the diagonal's
                              // imaginary part is kept (the original algorithm's full-gemm fold,
                              // pipeline.cpp:266-271, does not zero it); else forced to 0
  unsigned long long* stamp;  // optional launch timestamp slot (stamp.cuh); launch_tri_kernel gives
                              // its k-th kernel the slot stamp + k * kStampWords
  double alpha_re, alpha_im;
  double beta;             // real; 0 => C is never read
};

}  // namespace hsdla_b200
