// C++ drop-in adapter: the reference's own pipeline API on top of the hsdla_b200 C-ABI.
//
// Header-only; compiled inside the reference tree (it includes the reference's
// public headers, proj/include/hsdla/*.hpp) and linked against libhsdla_b200.so.
//
//   hsdla::pipeline::HSResult hsdla_b200::build_hs_refined(const hsdla::ProblemInstance&,
//                                                         const hsdla::pipeline::PipelineConfig&,
//                                                         const hsdla_b200::Options& = {})
// has the contract of hsdla::pipeline::build_hs_refined (pipeline.hpp:55,
// pipeline.cpp:281-329): fresh lower-authoritative H and S with exactly-zero upper
// triangles, diagonal imaginary parts 0, ledger == flop_model(p, Refined), five
// phases named s, z_loop, her2k, hemm_loop, herkx, peak_temp_bytes = the device
// temporaries.  hsdla_b200::build_hs_original has the contract of
// hsdla::pipeline::build_hs_original (pipeline.hpp:51, pipeline.cpp:189-279):
// ledger == flop_model(p, Original), phases z_loop, her2k, s, chol_loop,
// h_aa_update.  hsdla_b200::build_hs dispatches on cfg.variant (pipeline.cpp:331-334).  C-ABI status codes are rethrown as the reference's exception types
// (errors.hpp:9-26).  No CPU fallback: without a visible GPU it throws ConfigError.
#pragma once

#include <cstring>
#include <string>
#include <vector>

#include "hsdla/errors.hpp"
#include "hsdla/pipeline.hpp"
#include "hsdla/problem.hpp"
#include "hsdla_b200.h"

namespace hsdla_b200 {

struct Options {
  int n_gpus = 1;                             // GPUs: col_groups column windows x atom shards
  std::vector<int> device_ids;                // empty: 0..n_gpus-1
  int algo = HSDLA_B200_ALGO_REFINED_MERGED;  // or REFINED_FUSED, or REFINED (reference phase order)
  int arith = HSDLA_B200_ARITH_3M;            // or HSDLA_B200_ARITH_4M (plain 4-multiplication complex)
  bool reduce_to_root = false;                // true: ncclReduce onto device_ids[0]; false: reduce-scatter,
                                              // every GPU downloads its own slices
  int col_groups = 0;                         // 2-D tiling of H, S (0: automatic by memory budget)
  double mem_budget_gb = 0.0;                 // per-GPU budget of the automatic choice (0: 90 % of free)
};

inline void throw_status(int rc, const char* what) {
  if (rc == HSDLA_B200_OK) return;
  const std::string msg = std::string(what) + ": " + hsdla_b200_last_error();
  switch (rc) {
    case HSDLA_B200_DIMENSION_ERROR: throw hsdla::DimensionError(msg);
    case HSDLA_B200_SIZING_ERROR: throw hsdla::SizingError(msg);
    case HSDLA_B200_CONFIG_ERROR: throw hsdla::ConfigError(msg);
    case HSDLA_B200_IO_ERROR: throw hsdla::IoError(msg);
    default: throw std::runtime_error(msg);
  }
}

namespace detail {

inline hsdla_b200_options c_options(const Options& opt, int algo) {
  hsdla_b200_options co{};
  co.n_gpus = opt.n_gpus;
  co.device_ids = opt.device_ids.empty() ? nullptr : opt.device_ids.data();
  co.algo = algo;
  co.flags = (opt.arith == HSDLA_B200_ARITH_4M ? static_cast<int>(HSDLA_B200_FLAG_ARITH_4M) : 0) |
             (opt.reduce_to_root ? static_cast<int>(HSDLA_B200_FLAG_REDUCE_ROOT) : 0);
  co.col_groups = opt.col_groups;
  co.mem_budget_gb = opt.mem_budget_gb;
  return co;
}

// The algorithm a call runs: Original for Variant::Original, else opt.algo, which must then
// be one of the refined algorithms (build_hs_refined's check, pipeline.hpp:55).
inline int refined_algo(const Options& opt, const char* what) {
  if (opt.algo != HSDLA_B200_ALGO_REFINED_MERGED && opt.algo != HSDLA_B200_ALGO_REFINED_FUSED &&
      opt.algo != HSDLA_B200_ALGO_REFINED)
    throw hsdla::ConfigError(std::string(what) + ": algo must be REFINED_MERGED, REFINED_FUSED or REFINED");
  return opt.algo;
}
inline int algo_of(const hsdla::pipeline::PipelineConfig& cfg, const Options& opt, const char* what) {
  return cfg.variant == hsdla::pipeline::Variant::Original ? HSDLA_B200_ALGO_ORIGINAL : refined_algo(opt, what);
}

inline void fill_result(hsdla::pipeline::HSResult& r, const hsdla_b200_stats& st, int algo) {
  static const char* const keys[8] = {"gemm", "hemm", "her2k", "herk", "scaling", "herkx", "potrf", "trmm"};
  for (int i = 0; i < 8; ++i)
    if (st.ledger[i]) r.ledger.add(keys[i], st.ledger[i]);
  // reported phases in the reference's order, read from their slots
  static const int refined_slots[5] = {HSDLA_B200_PHASE_S, HSDLA_B200_PHASE_Z_LOOP, HSDLA_B200_PHASE_HER2K,
                                       HSDLA_B200_PHASE_HEMM_LOOP, HSDLA_B200_PHASE_HERKX};
  static const char* const refined_names[5] = {"s", "z_loop", "her2k", "hemm_loop", "herkx"};
  static const int original_slots[5] = {HSDLA_B200_PHASE_Z_LOOP, HSDLA_B200_PHASE_HER2K, HSDLA_B200_PHASE_S,
                                        HSDLA_B200_PHASE_CHOL_LOOP, HSDLA_B200_PHASE_H_AA_UPDATE};
  static const char* const original_names[5] = {"z_loop", "her2k", "s", "chol_loop", "h_aa_update"};
  const bool orig = algo == HSDLA_B200_ALGO_ORIGINAL;
  for (int i = 0; i < 5; ++i)
    r.phases.push_back({orig ? original_names[i] : refined_names[i],
                        st.phase_seconds[orig ? original_slots[i] : refined_slots[i]]});
  r.peak_temp_bytes = static_cast<std::size_t>(st.peak_temp_bytes);
  if (algo == HSDLA_B200_ALGO_REFINED_FUSED) r.warnings.push_back("herkx fused into the her2k contraction");
  if (algo == HSDLA_B200_ALGO_REFINED_MERGED)
    r.warnings.push_back("her2k, hemm_loop and herkx merged into one H contraction [A;B]^H [W_A;W_B]");
}

// The reference keeps each atom's operator blocks and U in separate heap blocks: pack them
// into the contiguous layout of the C-ABI.  pack_ops validates the operators and U only
// (the k-point batch does not use the cell's A, B); check_coefficients validates A, B.
struct PackedOps {
  std::vector<hsdla::cplx> taa, tab, tbb;
  std::vector<double> u;
};
inline void check_coefficients(const hsdla::ProblemInstance& p) {
  if (p.A.rows() != p.n_atoms * p.n_l || p.A.cols() != p.n_g || !p.A.same_shape(p.B))
    throw hsdla::DimensionError("build_hs: malformed ProblemInstance");
}
inline PackedOps pack_ops(const hsdla::ProblemInstance& p) {
  const std::size_t na = p.n_atoms, nl = p.n_l;
  if (p.T_AA.size() != na || p.T_AB.size() != na || p.T_BB.size() != na || p.U.size() != na)
    throw hsdla::DimensionError("build_hs: malformed ProblemInstance");
  const std::size_t blk = nl * nl;
  PackedOps o{std::vector<hsdla::cplx>(na * blk), std::vector<hsdla::cplx>(na * blk),
              std::vector<hsdla::cplx>(na * blk), std::vector<double>(na * nl)};
  std::vector<hsdla::cplx>&taa = o.taa, &tab = o.tab, &tbb = o.tbb;
  std::vector<double>& u = o.u;
  for (std::size_t a = 0; a < na; ++a) {
    if (p.T_AA[a].order() != nl || p.T_AB[a].rows() != nl || p.T_AB[a].cols() != nl ||
        p.T_BB[a].order() != nl || p.U[a].size() != nl)
      throw hsdla::DimensionError("build_hs: operator block of wrong order");
    std::memcpy(static_cast<void*>(taa.data() + a * blk), p.T_AA[a].matrix().data(), blk * sizeof(hsdla::cplx));
    std::memcpy(static_cast<void*>(tab.data() + a * blk), p.T_AB[a].data(), blk * sizeof(hsdla::cplx));
    std::memcpy(static_cast<void*>(tbb.data() + a * blk), p.T_BB[a].matrix().data(), blk * sizeof(hsdla::cplx));
    std::memcpy(u.data() + a * nl, p.U[a].data(), nl * sizeof(double));
  }
  return o;
}

inline hsdla::pipeline::HSResult run(const hsdla::ProblemInstance& p, int algo, const Options& opt) {
  const std::size_t na = p.n_atoms, nl = p.n_l, ng = p.n_g;
  check_coefficients(p);
  const PackedOps ops = pack_ops(p);
  const std::vector<hsdla::cplx>&taa = ops.taa, &tab = ops.tab, &tbb = ops.tbb;
  const std::vector<double>& u = ops.u;
  hsdla_b200_problem cp{na, nl, ng,
                        reinterpret_cast<const double*>(p.A.data()), reinterpret_cast<const double*>(p.B.data()),
                        reinterpret_cast<const double*>(taa.data()), reinterpret_cast<const double*>(tab.data()),
                        reinterpret_cast<const double*>(tbb.data()), u.data()};
  const hsdla_b200_options co = c_options(opt, algo);
  hsdla::pipeline::HSResult r;
  r.H = hsdla::HermitianView(ng);  // zero-initialised: the upper triangle stays exactly 0
  r.S = hsdla::HermitianView(ng);
  hsdla_b200_stats st{};
  throw_status(hsdla_b200_build_hs(&cp, &co, reinterpret_cast<double*>(r.H.matrix().data()),
                                   reinterpret_cast<double*>(r.S.matrix().data()), &st),
               "hsdla_b200_build_hs");
  fill_result(r, st, algo);
  return r;
}

}  // namespace detail

inline hsdla::pipeline::HSResult build_hs_refined(const hsdla::ProblemInstance& p,
                                                  const hsdla::pipeline::PipelineConfig& cfg,
                                                  const Options& opt = {}) {
  if (cfg.variant != hsdla::pipeline::Variant::Refined)
    throw hsdla::ConfigError("build_hs_refined: variant must be Refined");
  return detail::run(p, detail::refined_algo(opt, "build_hs_refined"), opt);
}

inline hsdla::pipeline::HSResult build_hs_original(const hsdla::ProblemInstance& p,
                                                   const hsdla::pipeline::PipelineConfig& /*cfg*/,
                                                   const Options& opt = {}) {
  return detail::run(p, HSDLA_B200_ALGO_ORIGINAL, opt);
}

/// build_hs(load_problem(path), cfg) with the HSDL v1 file (problem.cpp:144-243) streamed
/// shard by shard straight into HBM: no host ProblemInstance.  IoError on a missing,
/// malformed or truncated file (test_io.cpp:47-63).
inline hsdla::pipeline::HSResult build_hs_file(const std::string& path, const hsdla::pipeline::PipelineConfig& cfg,
                                               const Options& opt = {}) {
  const int algo = detail::algo_of(cfg, opt, "build_hs_file");
  uint64_t na = 0, nl = 0, ng = 0;
  throw_status(hsdla_b200_problem_file_info(path.c_str(), &na, &nl, &ng, nullptr), "hsdla_b200_problem_file_info");
  const hsdla_b200_options co = detail::c_options(opt, algo);
  hsdla::pipeline::HSResult r;
  r.H = hsdla::HermitianView(ng);
  r.S = hsdla::HermitianView(ng);
  hsdla_b200_stats st{};
  throw_status(hsdla_b200_build_hs_file(path.c_str(), &co, reinterpret_cast<double*>(r.H.matrix().data()),
                                        reinterpret_cast<double*>(r.S.matrix().data()), &st),
               "hsdla_b200_build_hs_file");
  detail::fill_result(r, st, algo);
  return r;
}

/// k-point batch (an extension beside the per-k-point drop-in; hsdla_b200_build_hs_kpoints):
/// `cell` supplies the k-independent operators and U (its A, B are not used and not checked),
/// As[k] / Bs[k] each k-point's coefficients ((n_atoms n_l) x N_G(k), as ProblemInstance::A / B;
/// N_G(k) may differ per k-point).  On one GPU the upload of k+1 and the download of k-1
/// overlap the build of k.  Same results as one build_hs per k-point, to FP64 rounding.
/// Ledgers are per k-point (flop_model at N_G(k)); phase times are the LAST k-point's device
/// times (the batch pipelines the k-points, so earlier ones have no separate phase record).
inline std::vector<hsdla::pipeline::HSResult> build_hs_kpoints(const hsdla::ProblemInstance& cell,
                                                               const std::vector<hsdla::ComplexMatrix>& As,
                                                               const std::vector<hsdla::ComplexMatrix>& Bs,
                                                               const hsdla::pipeline::PipelineConfig& cfg,
                                                               const Options& opt = {}) {
  const std::size_t na = cell.n_atoms, nl = cell.n_l, nk = As.size();
  if (Bs.size() != nk) throw hsdla::DimensionError("build_hs_kpoints: As and Bs differ in length");
  std::vector<uint64_t> ngk(nk);
  for (std::size_t k = 0; k < nk; ++k) {
    if (As[k].rows() != na * nl || As[k].cols() < 1 || !As[k].same_shape(Bs[k]))
      throw hsdla::DimensionError("build_hs_kpoints: k-point coefficients of wrong shape");
    ngk[k] = As[k].cols();
  }
  const int algo = detail::algo_of(cfg, opt, "build_hs_kpoints");
  const detail::PackedOps ops = detail::pack_ops(cell);
  hsdla_b200_problem cp{na, nl, nk ? ngk[0] : cell.n_g, nullptr, nullptr,
                        reinterpret_cast<const double*>(ops.taa.data()), reinterpret_cast<const double*>(ops.tab.data()),
                        reinterpret_cast<const double*>(ops.tbb.data()), ops.u.data()};
  const hsdla_b200_options co = detail::c_options(opt, algo);
  std::vector<hsdla::pipeline::HSResult> out(nk);
  std::vector<const double*> a(nk), b(nk);
  std::vector<double*> h(nk), s(nk);
  for (std::size_t k = 0; k < nk; ++k) {
    out[k].H = hsdla::HermitianView(ngk[k]);
    out[k].S = hsdla::HermitianView(ngk[k]);
    a[k] = reinterpret_cast<const double*>(As[k].data());
    b[k] = reinterpret_cast<const double*>(Bs[k].data());
    h[k] = reinterpret_cast<double*>(out[k].H.matrix().data());
    s[k] = reinterpret_cast<double*>(out[k].S.matrix().data());
  }
  if (nk == 0) return out;
  hsdla_b200_stats st{};
  throw_status(hsdla_b200_build_hs_kpoints(&cp, nk, ngk.data(), a.data(), b.data(), &co, h.data(), s.data(), &st),
               "hsdla_b200_build_hs_kpoints");
  for (std::size_t k = 0; k < nk; ++k) {
    hsdla_b200_stats sk = st;  // the ledger of k-point k (flop_model at N_G(k))
    throw_status(hsdla_b200_flop_model(algo == HSDLA_B200_ALGO_ORIGINAL ? 0 : 1, na, nl, ngk[k], st.n_hpd,
                                       sk.ledger),
                 "hsdla_b200_flop_model");
    detail::fill_result(out[k], sk, algo);
  }
  return out;
}

inline hsdla::pipeline::HSResult build_hs(const hsdla::ProblemInstance& p, const hsdla::pipeline::PipelineConfig& cfg,
                                          const Options& opt = {}) {
  return cfg.variant == hsdla::pipeline::Variant::Original ? build_hs_original(p, cfg, opt)
                                                           : build_hs_refined(p, cfg, opt);
}

}  // namespace hsdla_b200
