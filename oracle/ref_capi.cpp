// TEST INFRASTRUCTURE ONLY — not product code.
//
// extern "C" bridge over the UNMODIFIED reference library, compiled from the
// sources where they lie under /root/reference/proj/src by oracle/Makefile
// into oracle/_ref/libhsdla_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg / --impl reference) load it, as the checker or the
// CPU baseline — never as the measured or shipped path.
//
// Entry points mirror the reference API used on the hot path:
//   generate_problem   proj/src/problem.cpp:79-142
//   build_hs_refined   proj/src/pipeline.cpp:281-329 (Strategy::Cpu)
//   build_hs_original  proj/src/pipeline.cpp:189-279
//   flop_model         proj/src/pipeline.cpp:336-364
//   oracle::direct_*   proj/src/oracle.cpp:72-126
//   save/load_problem  proj/src/problem.cpp:172-243
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "hsdla/oracle.hpp"
#include "hsdla/pipeline.hpp"
#include "hsdla/problem.hpp"

using namespace hsdla;

namespace {

thread_local std::string g_err;

// Ledger keys in a fixed order shared with oracle/oracle.py.
const char* const kKeys[8] = {"gemm", "hemm", "her2k", "herk", "scaling", "herkx", "potrf", "trmm"};

void put_ledger(const FlopLedger& l, std::uint64_t* out) {
  for (int i = 0; i < 8; ++i) out[i] = l.count(kKeys[i]);
  out[8] = l.total();
}

void copy_cm(const ComplexMatrix& m, double* dst) {
  std::memcpy(dst, m.data(), m.size() * sizeof(cplx));
}

ProblemInstance make_problem(std::uint64_t na, std::uint64_t nl, std::uint64_t ng, const double* A,
                             const double* B, const double* taa, const double* tab,
                             const double* tbb, const double* u, const std::uint8_t* hpd) {
  ProblemInstance p;
  p.n_atoms = na;
  p.n_l = nl;
  p.n_g = ng;
  p.A = ComplexMatrix(na * nl, ng);
  p.B = ComplexMatrix(na * nl, ng);
  std::memcpy(p.A.data(), A, p.A.size() * sizeof(cplx));
  std::memcpy(p.B.data(), B, p.B.size() * sizeof(cplx));
  const std::size_t blk = nl * nl;
  for (std::size_t a = 0; a < na; ++a) {
    ComplexMatrix m1(nl, nl), m2(nl, nl), m3(nl, nl);
    std::memcpy(m1.data(), taa + 2 * a * blk, blk * sizeof(cplx));
    std::memcpy(m2.data(), tab + 2 * a * blk, blk * sizeof(cplx));
    std::memcpy(m3.data(), tbb + 2 * a * blk, blk * sizeof(cplx));
    p.T_AA.emplace_back(std::move(m1));
    p.T_AB.push_back(std::move(m2));
    p.T_BB.emplace_back(std::move(m3));
    p.U.emplace_back(u + a * nl, u + (a + 1) * nl);
    p.hpd_flags.push_back(hpd ? hpd[a] != 0 : true);
  }
  return p;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 1;
  } catch (const SizingError& e) {
    g_err = e.what();
    return 2;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Fills caller buffers (A, B: 2*na*nl*ng doubles; T*: 2*na*nl*nl; U: na*nl; hpd: na).
int ref_generate(std::uint64_t na, std::uint64_t nl, std::uint64_t ng, std::uint64_t seed,
                 std::uint64_t n_not_hpd, double* A, double* B, double* taa, double* tab,
                 double* tbb, double* u, std::uint8_t* hpd) {
  return guarded([&] {
    const ProblemInstance p = generate_problem(na, nl, ng, seed, n_not_hpd);
    copy_cm(p.A, A);
    copy_cm(p.B, B);
    const std::size_t blk = nl * nl;
    for (std::size_t a = 0; a < na; ++a) {
      copy_cm(p.T_AA[a].matrix(), taa + 2 * a * blk);
      copy_cm(p.T_AB[a], tab + 2 * a * blk);
      copy_cm(p.T_BB[a].matrix(), tbb + 2 * a * blk);
      std::memcpy(u + a * nl, p.U[a].data(), nl * sizeof(double));
      hpd[a] = p.hpd_flags[a] ? 1 : 0;
    }
  });
}

// variant: 0 original, 1 refined.  kernel_variant: 0 Reference, 1 BlockedParallel.
// H, S: full n_g x n_g column-major complex outputs (upper triangle as the
// reference leaves it: zero).  phases: up to 8 seconds values; ledger: 9 u64.
int ref_build_hs(int variant, std::uint64_t na, std::uint64_t nl, std::uint64_t ng, const double* A,
                 const double* B, const double* taa, const double* tab, const double* tbb,
                 const double* u, const std::uint8_t* hpd, int kernel_variant, std::uint64_t block,
                 int threads, double* H, double* S, double* phase_seconds, int* n_phases,
                 std::uint64_t* ledger, double* wall_seconds, std::uint64_t* peak_temp_bytes) {
  return guarded([&] {
    const ProblemInstance p = make_problem(na, nl, ng, A, B, taa, tab, tbb, u, hpd);
    pipeline::PipelineConfig cfg;
    cfg.variant = variant == 0 ? pipeline::Variant::Original : pipeline::Variant::Refined;
    cfg.strategy = pipeline::Strategy::Cpu;
    cfg.kernel.variant = kernel_variant ? kernels::Variant::BlockedParallel : kernels::Variant::Reference;
    cfg.kernel.block = block;
    cfg.kernel.threads = threads;
    const auto t0 = std::chrono::steady_clock::now();
    const pipeline::HSResult r = pipeline::build_hs(p, cfg);
    *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (H) copy_cm(r.H.matrix(), H);
    if (S) copy_cm(r.S.matrix(), S);
    *n_phases = static_cast<int>(r.phases.size());
    for (std::size_t i = 0; i < r.phases.size() && i < 8; ++i) phase_seconds[i] = r.phases[i].seconds;
    put_ledger(r.ledger, ledger);
    *peak_temp_bytes = r.peak_temp_bytes;
  });
}

// which: 0 direct_H, 1 direct_S, 2 direct_H_grouped.  out: full n_g x n_g.
int ref_direct(int which, std::uint64_t na, std::uint64_t nl, std::uint64_t ng, const double* A,
               const double* B, const double* taa, const double* tab, const double* tbb,
               const double* u, double* out) {
  return guarded([&] {
    const ProblemInstance p = make_problem(na, nl, ng, A, B, taa, tab, tbb, u, nullptr);
    const HermitianView h = which == 0   ? oracle::direct_H(p)
                            : which == 1 ? oracle::direct_S(p)
                                         : oracle::direct_H_grouped(p);
    copy_cm(h.matrix(), out);
  });
}

int ref_flop_model(int variant, std::uint64_t na, std::uint64_t nl, std::uint64_t ng,
                   std::uint64_t n_hpd, std::uint64_t* ledger) {
  return guarded([&] {
    ProblemInstance dims;
    dims.n_atoms = na;
    dims.n_l = nl;
    dims.n_g = ng;
    dims.hpd_flags.assign(na, false);
    for (std::size_t a = 0; a < n_hpd && a < na; ++a) dims.hpd_flags[a] = true;
    put_ledger(pipeline::flop_model(
                   dims, variant == 0 ? pipeline::Variant::Original : pipeline::Variant::Refined),
               ledger);
  });
}

// kernels::potrf (kernels.cpp:417-436) on one n x n block (lower read).  l: full
// n x n factor (upper 0) when it succeeds.  *pivot: -1 on success, else the failing pivot.
int ref_potrf(std::uint64_t n, const double* a, double* l, std::int64_t* pivot) {
  return guarded([&] {
    HermitianView h(n);
    std::memcpy(static_cast<void*>(h.matrix().data()), a, n * n * sizeof(cplx));
    const kernels::PotrfResult r = kernels::potrf(h);
    *pivot = r.ok() ? -1 : static_cast<std::int64_t>(r.pivot);
    std::memset(l, 0, n * n * sizeof(cplx));
    if (r.ok()) copy_cm(*r.factor, l);
  });
}

int ref_save_problem(const char* path, std::uint64_t na, std::uint64_t nl, std::uint64_t ng,
                     const double* A, const double* B, const double* taa, const double* tab,
                     const double* tbb, const double* u, const std::uint8_t* hpd) {
  return guarded([&] { save_problem(make_problem(na, nl, ng, A, B, taa, tab, tbb, u, hpd), path); });
}

}  // extern "C"
