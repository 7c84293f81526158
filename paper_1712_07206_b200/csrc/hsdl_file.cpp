// HSDL v1 problem files (reference problem.cpp:144-243) streamed straight into the
// engine's device buffers: header parse, then the shard's rows of every A / B column
// (of the engine's column window), its T_AA / T_AB / T_BB blocks and U, copied from a
// cached read-only mapping of the file (or pread) by the host pool into pinned staging
// slabs and on to HBM on the copy stream while the next slab is read.  No host
// ProblemInstance is built.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>

#include "engine.hpp"
#include "hsdl_file.hpp"
#include "host_pool.hpp"

namespace hsdla_b200 {

// ---------------------------------------------------------------------------
// HSDL v1 problem files (reference problem.cpp:144-243) streamed straight into
// the engine's device buffers: header parse, then the shard's rows of every
// A / B column, its T_AA / T_AB / T_BB blocks and U, read with pread() by a few
// host threads into a double-buffered pinned staging ring and copied to HBM on the
// copy stream while the next slab is read.  No host ProblemInstance is built.
// ---------------------------------------------------------------------------
static void pread_all(int fd, void* dst, size_t bytes, uint64_t off) {
  char* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = pread(fd, p, bytes, static_cast<off_t>(off));
    if (r <= 0) throw Fail{HSDLA_B200_IO_ERROR, "problem file truncated"};  // problem.cpp:157-160
    p += r;
    bytes -= static_cast<size_t>(r);
    off += static_cast<uint64_t>(r);
  }
}

// problem.cpp:197-225: magic "HSDL", version 1, dims, hpd bit flags; checked_total.
HsdlHeader read_hsdl_header(int fd, const char* path) {
  HsdlHeader h;
  char magic[4];
  uint32_t version = 0;
  uint64_t dims[3];
  pread_all(fd, magic, 4, 0);
  if (std::memcmp(magic, "HSDL", 4) != 0) throw Fail{HSDLA_B200_IO_ERROR, std::string("bad magic: ") + path};
  pread_all(fd, &version, 4, 4);
  if (version != 1) throw Fail{HSDLA_B200_IO_ERROR, "unsupported format version " + std::to_string(version)};
  pread_all(fd, dims, sizeof(dims), 8);
  h.na = dims[0];
  h.nl = dims[1];
  h.ng = dims[2];
  const uint64_t max = UINT64_MAX / 16 / 4;  // checked_total (problem.cpp:69-75)
  if (h.nl != 0 && h.na > max / h.nl) throw Fail{HSDLA_B200_SIZING_ERROR, "n_atoms * n_l overflows"};
  if (h.ng != 0 && h.na * h.nl > max / h.ng) throw Fail{HSDLA_B200_SIZING_ERROR, "problem allocation overflows"};
  const uint64_t nflag = (h.na + 7) / 8;
  std::vector<uint8_t> flags(nflag);
  if (nflag) pread_all(fd, flags.data(), nflag, 32);
  h.hpd.resize(h.na);
  for (uint64_t a = 0; a < h.na; ++a) h.hpd[a] = (flags[a / 8] >> (a % 8)) & 1u;
  const uint64_t KG = h.na * h.nl * h.ng * 16;
  h.off_A = 32 + nflag;
  h.off_B = h.off_A + KG;
  h.off_T = h.off_B + KG;
  h.off_U = h.off_T + h.na * 3 * h.nl * h.nl * 16;
  h.total = h.off_U + h.na * h.nl * 8;
  struct stat sb;
  if (fstat(fd, &sb) != 0 || static_cast<uint64_t>(sb.st_size) < h.total)
    throw Fail{HSDLA_B200_IO_ERROR, "problem file truncated"};
  return h;
}

int open_hsdl(const char* path) {
  if (!path) throw Fail{HSDLA_B200_IO_ERROR, "null path"};
  const int fd = open(path, O_RDONLY);
  if (fd < 0) throw Fail{HSDLA_B200_IO_ERROR, std::string("cannot open: ") + path};
  return fd;
}

// Read `n` pieces of `piece` bytes at offsets off0 + i*stride into dst (packed),
// split over up to 8 threads.
static void pread_pieces(int fd, char* dst, uint64_t off0, uint64_t stride, size_t piece, uint64_t n,
                         size_t dpitch) {
  const uint64_t bytes = piece * n;
  const unsigned nt = bytes < (size_t(8) << 20) ? 1u : std::min<unsigned>(HostPool::get().width(), static_cast<unsigned>(n));
  std::vector<Fail> errs(nt);
  std::vector<char> bad(nt, 0);
  HostPool::get().run(nt, [&](uint64_t t) {
    const uint64_t i0 = n * t / nt, i1 = n * (t + 1) / nt;
    try {
      if (stride == piece && dpitch == piece) {
        pread_all(fd, dst + i0 * piece, (i1 - i0) * piece, off0 + i0 * stride);
      } else {
        for (uint64_t i = i0; i < i1; ++i) pread_all(fd, dst + i * dpitch, piece, off0 + i * stride);
      }
    } catch (const Fail& f) {
      errs[t] = f;
      bad[t] = 1;
    }
  });
  for (unsigned t = 0; t < nt; ++t)
    if (bad[t]) throw errs[t];
}

// The engine's cached read-only view of the open file `fd` (nullptr: mapping unavailable,
// the caller preads).  A different or changed file (device, inode, size, mtime) is
// remapped; MAP_POPULATE faults the page-cache pages in once per mapping.  The file
// must not be truncated while a call reads it (as for any mapped reader).
static const char* file_view(hsdla_b200_engine* e, int fd) {
  struct stat st {};
  if (fstat(fd, &st) != 0 || st.st_size <= 0) return nullptr;
  if (e->fmap && st.st_dev == e->fmap_st.st_dev && st.st_ino == e->fmap_st.st_ino &&
      st.st_size == e->fmap_st.st_size && st.st_mtim.tv_sec == e->fmap_st.st_mtim.tv_sec &&
      st.st_mtim.tv_nsec == e->fmap_st.st_mtim.tv_nsec)
    return e->fmap;
  if (e->fmap) munmap(const_cast<char*>(e->fmap), e->fmap_len);
  e->fmap = nullptr;
  void* m = mmap(nullptr, static_cast<size_t>(st.st_size), PROT_READ, MAP_SHARED | MAP_POPULATE, fd, 0);
  if (m == MAP_FAILED) return nullptr;
  e->fmap = static_cast<const char*>(m);
  e->fmap_len = static_cast<size_t>(st.st_size);
  e->fmap_st = st;
  return e->fmap;
}

// pread_pieces through the file view when there is one: copy_nt from the mapped page cache
// on the host pool (no syscall per piece)
static void read_pieces(hsdla_b200_engine* e, const char* view, int fd, char* dst, uint64_t off0, uint64_t stride,
                        size_t piece, uint64_t n, size_t dpitch = 0) {
  if (!dpitch) dpitch = piece;
  if (!view) {
    pread_pieces(fd, dst, off0, stride, piece, n, dpitch);
    return;
  }
  if (n && off0 + (n - 1) * stride + piece > e->fmap_len) throw Fail{HSDLA_B200_IO_ERROR, "truncated problem file"};
  par_for(n, n * piece, [&](uint64_t i) { copy_nt(dst + i * dpitch, view + off0 + i * stride, piece); });
  _mm_sfence();
}

// Host-read + H2D (on stream s) of the engine-local atoms [b0, b1) of shard a0 of an
// HSDL file: their rows of every A / B column (one pread per column when the rows
// are a strict subset of the file's, else whole column slabs), their T blocks and U.
static void load_atoms_from_file(hsdla_b200_engine* e, int fd, const HsdlHeader& h, uint64_t a0, uint64_t b0,
                                 uint64_t b1, cudaStream_t s) {
  const uint64_t K = e->K, Kf = h.na * h.nl, nl = h.nl, ng = h.ng - e->c0;  // the window's columns [c0, N_G)
  const uint64_t r0 = b0 * nl, rows = (b1 - b0) * nl, g0 = (a0 + b0) * nl + e->c0 * Kf;
  const size_t colb = rows * sizeof(double2);
  const char* view = file_view(e, fd);
  for (int m = 0; m < 2; ++m) {  // A then B
    const uint64_t base = (m == 0 ? h.off_A : h.off_B) + g0 * 16;
    double2* dst = (m == 0 ? e->A(0) : e->B(0)) + r0;
    if (colb > kStageSlab) {  // one column's rows exceed a slab: split the rows
      for (uint64_t j = 0; j < ng; ++j)
        for (uint64_t q0 = 0; q0 < rows; q0 += kStageSlab / 16) {
          const uint64_t nr = std::min<uint64_t>(kStageSlab / 16, rows - q0);
          int slot;
          char* b = stage_acquire(e, slot);
          read_pieces(e, view, fd, b, base + (j * Kf + q0) * 16, nr * 16, nr * 16, 1);
          HS_CUDA(cudaMemcpyAsync(dst + j * K + q0, b, nr * 16, cudaMemcpyHostToDevice, s));
          stage_release(e, slot, s);
        }
      continue;
    }
    const size_t sp = colb == Kf * 16 ? colb : slab_pitch(colb);  // 4 KB-aligned rows (engine.hpp)
    const uint64_t cols = std::max<uint64_t>(1, kStageSlab / sp);
    for (uint64_t j0 = 0; j0 < ng; j0 += cols) {
      const uint64_t nc = std::min(cols, ng - j0);
      int slot;
      char* b = stage_acquire(e, slot);
      read_pieces(e, view, fd, b, base + j0 * Kf * 16, Kf * 16, colb, nc, sp);
      HS_CUDA(cudaMemcpy2DAsync(dst + j0 * K, K * sizeof(double2), b, sp, colb, nc, cudaMemcpyHostToDevice, s));
      stage_release(e, slot, s);
    }
  }
  // operator blocks: T_AA, T_AB, T_BB interleaved per atom in the file
  const uint64_t blk = nl * nl * 16;
  if (3 * blk > kStageSlab) throw Fail{HSDLA_B200_SIZING_ERROR, "operator block larger than the staging slab"};
  const uint64_t atoms_per = std::max<uint64_t>(1, kStageSlab / (3 * blk));
  for (uint64_t c0 = b0; c0 < b1; c0 += atoms_per) {
    const uint64_t nb = std::min(atoms_per, b1 - c0);
    int slot;
    char* b = stage_acquire(e, slot);
    read_pieces(e, view, fd, b, h.off_T + (a0 + c0) * 3 * blk, 3 * blk, 3 * blk, nb);
    double2* dsts[3] = {e->Taa, e->Tab, e->Tbb};
    for (int m = 0; m < 3; ++m)
      HS_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(dsts[m]) + c0 * blk, blk, b + m * blk, 3 * blk, blk, nb,
                                cudaMemcpyHostToDevice, s));
    stage_release(e, slot, s);
  }
  const size_t ub = rows * sizeof(double);
  if (ub > kStageSlab) throw Fail{HSDLA_B200_SIZING_ERROR, "U larger than the staging slab"};
  int slot;
  char* b = stage_acquire(e, slot);
  read_pieces(e, view, fd, b, h.off_U + (a0 + b0) * nl * sizeof(double), ub, ub, 1);
  HS_CUDA(cudaMemcpyAsync(e->U + r0, b, ub, cudaMemcpyHostToDevice, s));
  stage_release(e, slot, s);
}

static HsdlHeader open_shard(Fd& f, const char* path, const hsdla_b200_engine* e, uint64_t a0) {
  f.fd = open_hsdl(path);
  HsdlHeader h = read_hsdl_header(f.fd, path);
  if (h.nl != e->nl || h.ng != e->ng || a0 + e->na > h.na)
    throw Fail{HSDLA_B200_DIMENSION_ERROR, "problem file shape does not match the engine shard"};
  return h;
}

void engine_load_file(hsdla_b200_engine* e, const char* path, uint64_t a0) {
  Fd f;
  const HsdlHeader h = open_shard(f, path, e, a0);
  HS_CUDA(cudaSetDevice(e->device));
  cudaStream_t s = e->copy_stream;
  // nothing may overwrite A/B/T/U while a previous build still reads them
  HS_CUDA(cudaStreamWaitEvent(s, e->ev_end, 0));
  load_atoms_from_file(e, f.fd, h, a0, 0, e->na, s);
  HS_CUDA(cudaEventRecord(e->ev_up1, s));
  HS_CUDA(cudaStreamWaitEvent(e->stream, e->ev_up1, 0));
}

// Streamed build from an HSDL file: the host reads atom chunk c+1 from the file
// while the GPU computes chunk c (the streamed chunk plans of the host-buffer path).
void engine_build_file(hsdla_b200_engine* e, const char* path, uint64_t a0, int algo) {
  Fd f;
  const HsdlHeader h = open_shard(f, path, e, a0);
  begin_build(e, algo);
  ensure_streamed_plans(e);
  copy_after_compute(e);  // the previous build (and any upload on the compute stream) is done with A, B, T, U
  HS_CUDA(cudaEventRecord(e->ev_up0, e->copy_stream));
  // the mapped file view feeds ~36-42 GB/s (copy_nt from the page cache): the host-packed
  // plan; HSDLA_B200_FILE_PLAN=pinned selects the page-locked one
  const char* fpl = std::getenv("HSDLA_B200_FILE_PLAN");
  auto& plan = fpl && std::strcmp(fpl, "pinned") == 0 ? e->streamed : e->streamed_pg;
  for (size_t c = 0; c < plan.size(); ++c) {
    load_atoms_from_file(e, f.fd, h, a0, plan[c].a0, plan[c].a1, e->copy_stream);
    HS_CUDA(cudaEventRecord(e->ev_chunk_up[c], e->copy_stream));
    HS_CUDA(cudaStreamWaitEvent(e->stream, e->ev_chunk_up[c], 0));
    if (c == 0) mark_build_begin(e);
    enqueue_chunk(e, plan[c], algo, c + 1 == plan.size(), nullptr);
  }
  HS_CUDA(cudaEventRecord(e->ev_up1, e->copy_stream));
  mark_build_end(e);
  e->uploaded_streamed = true;
}

void release_file_view(hsdla_b200_engine* e) {
  if (e->fmap) munmap(const_cast<char*>(e->fmap), e->fmap_len);
  e->fmap = nullptr;
  e->fmap_len = 0;
}

}  // namespace hsdla_b200
