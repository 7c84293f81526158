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
// temporaries.  C-ABI status codes are rethrown as the reference's exception types
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
  int n_gpus = 1;                             // atoms sharded over n_gpus, NCCL reduce to device_ids[0]
  std::vector<int> device_ids;                // empty: 0..n_gpus-1
  int algo = HSDLA_B200_ALGO_REFINED_FUSED;   // or HSDLA_B200_ALGO_REFINED (reference phase order)
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

inline hsdla::pipeline::HSResult build_hs_refined(const hsdla::ProblemInstance& p,
                                                  const hsdla::pipeline::PipelineConfig& cfg,
                                                  const Options& opt = {}) {
  if (cfg.variant != hsdla::pipeline::Variant::Refined)
    throw hsdla::ConfigError("hsdla_b200 implements the refined variant (Algorithm 3)");
  const std::size_t na = p.n_atoms, nl = p.n_l, ng = p.n_g;
  if (p.A.rows() != na * nl || p.A.cols() != ng || !p.A.same_shape(p.B) || p.T_AA.size() != na ||
      p.T_AB.size() != na || p.T_BB.size() != na || p.U.size() != na)
    throw hsdla::DimensionError("build_hs_refined: malformed ProblemInstance");
  // per-atom operator blocks are separate heap blocks in the reference: pack them
  const std::size_t blk = nl * nl;
  std::vector<hsdla::cplx> taa(na * blk), tab(na * blk), tbb(na * blk);
  std::vector<double> u(na * nl);
  for (std::size_t a = 0; a < na; ++a) {
    if (p.T_AA[a].order() != nl || p.T_AB[a].rows() != nl || p.T_AB[a].cols() != nl ||
        p.T_BB[a].order() != nl || p.U[a].size() != nl)
      throw hsdla::DimensionError("build_hs_refined: operator block of wrong order");
    std::memcpy(taa.data() + a * blk, p.T_AA[a].matrix().data(), blk * sizeof(hsdla::cplx));
    std::memcpy(tab.data() + a * blk, p.T_AB[a].data(), blk * sizeof(hsdla::cplx));
    std::memcpy(tbb.data() + a * blk, p.T_BB[a].matrix().data(), blk * sizeof(hsdla::cplx));
    std::memcpy(u.data() + a * nl, p.U[a].data(), nl * sizeof(double));
  }
  hsdla_b200_problem cp{na, nl, ng,
                        reinterpret_cast<const double*>(p.A.data()), reinterpret_cast<const double*>(p.B.data()),
                        reinterpret_cast<const double*>(taa.data()), reinterpret_cast<const double*>(tab.data()),
                        reinterpret_cast<const double*>(tbb.data()), u.data()};
  hsdla_b200_options co{opt.n_gpus, opt.device_ids.empty() ? nullptr : opt.device_ids.data(), opt.algo, 0};
  hsdla::pipeline::HSResult r;
  r.H = hsdla::HermitianView(ng);  // zero-initialised: the upper triangle stays exactly 0
  r.S = hsdla::HermitianView(ng);
  hsdla_b200_stats st{};
  throw_status(hsdla_b200_build_hs(&cp, &co, reinterpret_cast<double*>(r.H.matrix().data()),
                                   reinterpret_cast<double*>(r.S.matrix().data()), &st),
               "hsdla_b200_build_hs");
  static const char* const keys[8] = {"gemm", "hemm", "her2k", "herk", "scaling", "herkx", "potrf", "trmm"};
  for (int i = 0; i < 8; ++i)
    if (st.ledger[i]) r.ledger.add(keys[i], st.ledger[i]);
  static const char* const phases[5] = {"s", "z_loop", "her2k", "hemm_loop", "herkx"};
  for (int i = 0; i < 5; ++i) r.phases.push_back({phases[i], st.phase_seconds[i]});
  r.peak_temp_bytes = static_cast<std::size_t>(st.peak_temp_bytes);
  if (opt.algo == HSDLA_B200_ALGO_REFINED_FUSED) r.warnings.push_back("herkx fused into the her2k contraction");
  return r;
}

inline hsdla::pipeline::HSResult build_hs(const hsdla::ProblemInstance& p, const hsdla::pipeline::PipelineConfig& cfg,
                                          const Options& opt = {}) {
  if (cfg.variant == hsdla::pipeline::Variant::Original)
    throw hsdla::ConfigError("hsdla_b200: the original variant (Algorithm 1) is not provided");
  return build_hs_refined(p, cfg, opt);
}

}  // namespace hsdla_b200
