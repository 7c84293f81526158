// TEST INFRASTRUCTURE ONLY — C++ drop-in parity driver.
//
// Links the UNMODIFIED reference library (oracle/_ref/libhsdla_ref.so, built from
// /root/reference/proj/src) and libhsdla_b200.so, and drives BOTH through the
// reference's own C++ types: hsdla::generate_problem -> hsdla::pipeline::build_hs_refined /
// build_hs(Original) (CPU) vs hsdla_b200::build_hs_refined / build_hs (include/hsdla_b200/
// pipeline.hpp, GPU).
// Exit code = number of failed checks (the acceptance.cpp convention).
//   parity_cpp <n_atoms> <n_l> <n_g> <seed> <n_not_hpd> [threads]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <cstdio>
#include <cstdlib>

#include "hsdla/pipeline.hpp"
#include "hsdla/problem.hpp"
#include "hsdla_b200/kernels.hpp"
#include "hsdla_b200/pipeline.hpp"

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s n_atoms n_l n_g seed n_not_hpd [threads]\n", argv[0]);
    return 64;
  }
  const std::size_t na = std::atoll(argv[1]), nl = std::atoll(argv[2]), ng = std::atoll(argv[3]);
  const std::uint64_t seed = std::atoll(argv[4]);
  const std::size_t nnh = std::atoll(argv[5]);
  const int threads = argc > 6 ? std::atoi(argv[6]) : 0;
  const hsdla::ProblemInstance p = hsdla::generate_problem(na, nl, ng, seed, nnh);
  hsdla::pipeline::PipelineConfig cfg;
  cfg.kernel = {hsdla::kernels::Variant::BlockedParallel, 128, threads};
  const hsdla::pipeline::HSResult cpu = hsdla::pipeline::build_hs_refined(p, cfg);
  int fails = 0;
  auto check = [&](bool ok, const char* what, double v) {
    std::printf("%-44s %s (%.3e)\n", what, ok ? "PASS" : "FAIL", v);
    if (!ok) ++fails;
  };
  for (int algo : {HSDLA_B200_ALGO_REFINED_MERGED, HSDLA_B200_ALGO_REFINED_FUSED, HSDLA_B200_ALGO_REFINED,
                   HSDLA_B200_ALGO_REFINED_MERGED + 100, HSDLA_B200_ALGO_REFINED_FUSED + 100}) {
    hsdla_b200::Options opt;
    opt.arith = algo >= 100 ? HSDLA_B200_ARITH_4M : HSDLA_B200_ARITH_3M;  // +100: the same algorithm in 4M
    algo %= 100;
    opt.algo = algo;
    const hsdla::pipeline::HSResult gpu = hsdla_b200::build_hs_refined(p, cfg, opt);
    const double eh = hsdla::rel_frobenius_error_lower(gpu.H.matrix(), cpu.H.matrix());
    const double es = hsdla::rel_frobenius_error_lower(gpu.S.matrix(), cpu.S.matrix());
    std::printf("algo %d arith %s\n", algo, opt.arith == HSDLA_B200_ARITH_4M ? "4M" : "3M");
    check(eh <= 1e-11, "  H rel Frobenius (lower) <= 1e-11", eh);
    check(es <= 1e-11, "  S rel Frobenius (lower) <= 1e-11", es);
    check(gpu.ledger == hsdla::pipeline::flop_model(p, hsdla::pipeline::Variant::Refined),
          "  ledger == flop_model(p, Refined)", double(gpu.ledger.total()));
    check(gpu.ledger == cpu.ledger, "  ledger == reference CPU ledger", double(cpu.ledger.total()));
    bool upper0 = true, diag0 = true;
    for (std::size_t j = 0; j < ng; ++j) {
      diag0 = diag0 && gpu.H(j, j).imag() == 0.0 && gpu.S(j, j).imag() == 0.0;
      for (std::size_t i = 0; i < j; ++i)
        upper0 = upper0 && gpu.H(i, j) == hsdla::cplx(0.0) && gpu.S(i, j) == hsdla::cplx(0.0);
    }
    check(upper0, "  upper triangles exactly 0", 0.0);
    check(diag0, "  diagonal imaginary parts exactly 0", 0.0);
    bool names = gpu.phases.size() == 5;
    for (std::size_t i = 0; names && i < 5; ++i) names = gpu.phases[i].name == cpu.phases[i].name;
    check(names, "  phase names == reference", double(gpu.phases.size()));
  }
  // the original variant (Algorithm 1) through build_hs dispatch vs the reference's own
  // build_hs_original on the same instance
  {
    hsdla::pipeline::PipelineConfig ocfg = cfg;
    ocfg.variant = hsdla::pipeline::Variant::Original;
    const hsdla::pipeline::HSResult cpu_o = hsdla::pipeline::build_hs(p, ocfg);
    const hsdla::pipeline::HSResult gpu = hsdla_b200::build_hs(p, ocfg);
    const double eh = hsdla::rel_frobenius_error_lower(gpu.H.matrix(), cpu_o.H.matrix());
    const double es = hsdla::rel_frobenius_error_lower(gpu.S.matrix(), cpu_o.S.matrix());
    std::printf("variant original\n");
    check(eh <= 1e-11, "  H rel Frobenius (lower) <= 1e-11", eh);
    check(es <= 1e-11, "  S rel Frobenius (lower) <= 1e-11", es);
    check(gpu.ledger == hsdla::pipeline::flop_model(p, hsdla::pipeline::Variant::Original),
          "  ledger == flop_model(p, Original)", double(gpu.ledger.total()));
    check(gpu.ledger == cpu_o.ledger, "  ledger == reference CPU ledger", double(cpu_o.ledger.total()));
    bool names = gpu.phases.size() == cpu_o.phases.size();
    for (std::size_t i = 0; names && i < gpu.phases.size(); ++i) names = gpu.phases[i].name == cpu_o.phases[i].name;
    check(names, "  phase names == reference", double(gpu.phases.size()));
    bool upper0 = true;
    for (std::size_t j = 0; j < ng; ++j)
      for (std::size_t i = 0; i < j; ++i)
        upper0 = upper0 && gpu.H(i, j) == hsdla::cplx(0.0) && gpu.S(i, j) == hsdla::cplx(0.0);
    check(upper0, "  upper triangles exactly 0", 0.0);
  }
  // k-point batch (extension): three k-points of the cell, the first being p's own coefficients;
  // each equals the reference CPU run on that k-point's problem
  {
    std::vector<hsdla::ComplexMatrix> As{p.A}, Bs{p.B};
    std::vector<hsdla::ProblemInstance> kp;
    for (uint64_t k = 1; k < 3; ++k) {
      kp.push_back(hsdla::generate_problem(na, nl, ng, seed + 100 + k, nnh));
      As.push_back(kp.back().A);
      Bs.push_back(kp.back().B);
    }
    const auto got = hsdla_b200::build_hs_kpoints(p, As, Bs, cfg);
    std::printf("build_hs_kpoints (3 k-points)\n");
    double worst = 0.0;
    for (std::size_t k = 0; k < 3; ++k) {
      hsdla::ProblemInstance pk = p;
      pk.A = As[k];
      pk.B = Bs[k];
      const hsdla::pipeline::HSResult ref = k == 0 ? cpu : hsdla::pipeline::build_hs_refined(pk, cfg);
      worst = std::max({worst, hsdla::rel_frobenius_error_lower(got[k].H.matrix(), ref.H.matrix()),
                        hsdla::rel_frobenius_error_lower(got[k].S.matrix(), ref.S.matrix())});
    }
    check(got.size() == 3 && worst <= 1e-11, "  every k-point: H, S rel Frobenius (lower) <= 1e-11", worst);
  }
  // HSDL v1 file written by the reference's save_problem, streamed into HBM by the drop-in
  {
    const std::string path = "/tmp/hsdla_b200_parity_cpp.hsdl";
    hsdla::save_problem(p, path);
    const hsdla::pipeline::HSResult gpu = hsdla_b200::build_hs_file(path, cfg);
    const double eh = hsdla::rel_frobenius_error_lower(gpu.H.matrix(), cpu.H.matrix());
    const double es = hsdla::rel_frobenius_error_lower(gpu.S.matrix(), cpu.S.matrix());
    std::printf("build_hs_file\n");
    check(eh <= 1e-11 && es <= 1e-11, "  H, S rel Frobenius (lower) <= 1e-11", std::max(eh, es));
    check(gpu.ledger == cpu.ledger, "  ledger == reference CPU ledger", double(cpu.ledger.total()));
    std::remove(path.c_str());
    try {
      hsdla_b200::build_hs_file("/nonexistent/nowhere.hsdl", cfg);
      check(false, "  missing file -> IoError", 0);
    } catch (const hsdla::IoError&) {
      check(true, "  missing file -> IoError", 0);
    }
  }
  // the kernel layer (hsdla::kernels) against the reference's own CPU kernels on the same data
  {
    namespace rk = hsdla::kernels;
    namespace gk = hsdla_b200::kernels;
    const std::size_t kk = std::min<std::size_t>(na * nl, 300), n = std::min<std::size_t>(ng, 200);
    hsdla::ComplexMatrix a(kk, n), b(kk, n);
    for (std::size_t j = 0; j < n; ++j)
      for (std::size_t i = 0; i < kk; ++i) {
        a(i, j) = p.A(i, j);
        b(i, j) = p.B(i, j);
      }
    auto rel_lower = [&](const hsdla::HermitianView& x, const hsdla::HermitianView& y) {
      return hsdla::rel_frobenius_error_lower(x.matrix(), y.matrix());
    };
    const hsdla::cplx alpha(0.75, -0.5);
    hsdla::FlopLedger lc, lg;
    hsdla::HermitianView c1(n), c2(n);
    rk::herk(1.5, a, 0.0, c1, &lc);
    gk::herk(1.5, a, 0.0, c2, &lg);
    check(rel_lower(c2, c1) <= 1e-13, "kernels::herk vs reference", rel_lower(c2, c1));
    rk::her2k(alpha, a, b, 1.0, c1, &lc);
    gk::her2k(alpha, a, b, 1.0, c2, &lg);
    check(rel_lower(c2, c1) <= 1e-13, "kernels::her2k (beta 1) vs reference", rel_lower(c2, c1));
    rk::herkx(alpha, a, b, 0.5, c1, &lc);
    gk::herkx(alpha, a, b, 0.5, c2, &lg);
    check(rel_lower(c2, c1) <= 1e-13, "kernels::herkx (beta 1/2) vs reference", rel_lower(c2, c1));
    hsdla::ComplexMatrix g1(n, n), g2(n, n);
    rk::gemm(alpha, a, rk::Trans::ConjTrans, b, rk::Trans::None, hsdla::cplx(0.0), g1, &lc);
    gk::gemm(alpha, a, rk::Trans::ConjTrans, b, rk::Trans::None, hsdla::cplx(0.0), g2, &lg);
    check(hsdla::rel_frobenius_error_lower(g2, g1) <= 1e-13, "kernels::gemm vs reference",
          hsdla::rel_frobenius_error_lower(g2, g1));
    const hsdla::HermitianView& t = p.T_AA[0];
    hsdla::ComplexMatrix bs(nl, n), h1(nl, n), h2(nl, n);
    for (std::size_t j = 0; j < n; ++j)
      for (std::size_t i = 0; i < nl; ++i) bs(i, j) = p.B(i, j);
    rk::hemm(rk::Side::Left, alpha, t, bs, hsdla::cplx(0.0), h1, &lc);
    gk::hemm(rk::Side::Left, alpha, t, bs, hsdla::cplx(0.0), h2, &lg);
    double eh = 0, nh = 0;
    for (std::size_t i = 0; i < h1.size(); ++i) {
      eh += std::norm(h2.data()[i] - h1.data()[i]);
      nh += std::norm(h1.data()[i]);
    }
    check(std::sqrt(eh / nh) <= 1e-13, "kernels::hemm vs reference", std::sqrt(eh / nh));
    const auto f1 = rk::potrf(t, &lc), f2 = gk::potrf(t, &lg);
    bool same = f1.ok() == f2.ok();
    if (same && f1.ok())
      for (std::size_t i = 0; i < f1.factor->size(); ++i) same = same && f1.factor->data()[i] == f2.factor->data()[i];
    check(same, "kernels::potrf bit-identical to reference", 0.0);
    check(lg == lc, "kernel-layer ledger == reference ledger", double(lc.total()));
  }
  // error mapping: a refined call with a non-refined variant -> hsdla::ConfigError
  try {
    hsdla::pipeline::PipelineConfig bad = cfg;
    bad.variant = hsdla::pipeline::Variant::Original;
    hsdla_b200::build_hs_refined(p, bad);
    check(false, "build_hs_refined(Original) -> ConfigError", 0);
  } catch (const hsdla::ConfigError&) {
    check(true, "build_hs_refined(Original) -> ConfigError", 0);
  }
  std::printf("%d failure(s)\n", fails);
  return fails;
}
