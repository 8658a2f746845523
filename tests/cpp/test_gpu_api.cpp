// C++ API checks of ncstomo_gpu.hpp, restating reference doctest cases
// (proj/tests/unit/test_ops.cpp, test_circulant.cpp, test_solvers.cpp) against
// the GPU path.  Prints one line per case; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "ncstomo_gpu.hpp"

using namespace ncstomo_gpu;

static int failures = 0;
#define CHECK(cond, name)                                      \
  do {                                                         \
    bool ok_ = (cond);                                         \
    std::printf("%s %s\n", ok_ ? "PASS" : "FAIL", name);       \
    if (!ok_) ++failures;                                      \
  } while (0)

static std::vector<double> randn(std::size_t n, unsigned seed) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> d;
  std::vector<double> v(n);
  for (auto& x : v) x = d(g);
  return v;
}

int main() {
  // test_ops.cpp:16-24
  CHECK(default_detector_count(64) == 93 && default_detector_count(512) == 727,
        "default_detector_count");
  // test_ops.cpp:26-30
  bool threw = false;
  try {
    RadonMap bad(64, 60, 92);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw, "RadonMap rejects even detector count");
  // test_ops.cpp:32-35 (fp32 device arithmetic: 1e-5)
  {
    RadonMap r(64, 60, 93);
    auto x = randn(r.domain_size(), 123), u = randn(r.range_size(), 124);
    std::vector<double> ax(r.range_size()), atu(r.domain_size());
    r.forward(x, ax);
    r.adjoint(u, atu);
    double l = std::inner_product(ax.begin(), ax.end(), u.begin(), 0.0);
    double rr = std::inner_product(x.begin(), x.end(), atu.begin(), 0.0);
    CHECK(std::abs(l - rr) / std::max(1.0, std::abs(l)) <= 1e-5, "Radon adjoint probe");
  }
  // test_ops.cpp:37-47
  {
    RadonMap r(64, 48, 93);
    std::vector<double> x(r.domain_size(), 0.0), s(r.range_size());
    x[32 * 64 + 32] = 1.0;
    r.forward(x, s);
    bool ok = true;
    for (int t = 0; t < 48; ++t) {
      double tot = 0;
      for (int d = 0; d < 93; ++d) tot += s[t * 93 + d];
      ok = ok && std::abs(tot - 1.0) <= 0.05;
    }
    CHECK(ok, "impulse projects to ~1 per angle");
  }
  // test_ops.cpp:60-79
  {
    GradMap gm(3);
    std::vector<double> x = {1, 2, 4, 8, 16, 32, 64, 128, 256}, g(gm.range_size());
    gm.forward(x, g);
    CHECK(g[0] == -1 && g[1] == -2 && g[2] == -8 && g[5] == -128 && g[6] == -7 &&
              g[11] == 32 - 256,
          "gradient hand values");
  }
  // test_circulant.cpp:55-64: identity mask
  {
    int n = 16;
    SpectralMask one(n);
    for (auto& h : one.h) h = 1.0;
    auto x = randn(n * n, 5);
    std::vector<double> y(n * n);
    MaskApplier(n).apply(one, x, y);
    double e = 0;
    for (int i = 0; i < n * n; ++i) e = std::max(e, std::abs(y[i] - x[i]));
    CHECK(e < 1e-5, "identity mask");
  }
  // test_solvers.cpp:192-203 and 607-625 on a 32^2 CT problem
  {
    int n = 32, A = 24, D = default_detector_count(n);
    RadonMap geom(n, A, D);
    auto truth = randn(geom.domain_size(), 9);
    for (auto& v : truth) v = std::max(0.0, v);
    std::vector<double> sino(geom.range_size());
    geom.forward(truth, sino);
    ModelParams p;
    p.alpha = p.beta = 0.1;
    p.lambda = 0.01;
    SplitProblem prob = assemble_problem(sino, geom, p);
    SolverConfig cfg;
    cfg.alpha = p.alpha;
    cfg.gamma = 400.0;
    cfg.mask = metric_mask(radon_mask(n, 100.0, 400.0), p);
    SolverState s = make_state(prob);
    ncs_step(s, prob, cfg);
    bool ok = true;
    for (double v : s.x.v) ok = ok && v == 0.0;
    for (std::size_t i = 0; i < sino.size(); ++i)
      ok = ok && std::abs(s.u[i] + p.alpha * sino[i] / (1 + p.alpha)) <=
                     1e-6 * (1 + std::abs(sino[i]));
    CHECK(ok, "first step KAT");
    SolverState a = make_state(prob);
    for (int k = 0; k < 5; ++k) ncs_step(a, prob, cfg);
    cfg.max_iters = 5;
    cfg.record_every = 5;
    SolveResult r = ncs_solve(prob, cfg);
    CHECK(r.state.x.v == a.x.v && r.state.u == a.u, "ncs_solve(5) == 5 x ncs_step (bitwise)");
    CHECK(r.record.rows.size() == 2 && r.record.rows.back().iter == 5 && r.state.iter == 5,
          "record rows, final state iter");
    // divergence (test_solvers.cpp:627-644)
    SolverConfig bad;
    bad.alpha = p.alpha;
    bad.gamma = 1e-6;
    bad.max_iters = 3000;
    bad.record_every = 500;
    bool div = false;
    try {
      pdhg_solve(prob, bad);
    } catch (const DivergenceError& e) {
      div = e.iter > 0;
    }
    CHECK(div, "DivergenceError with iteration");
  }
  // GPU setup path (circulant.cpp:142-169, pipeline.cpp:100-110) and the
  // step-condition screen (solvers.cpp:206-245, 278).
  {
    int n = 32, A = 24, D = default_detector_count(n);
    RadonMap geom(n, A, D);
    const double dc = dc_response(geom);
    const double scale = calibrate_scale(geom, 8, 0);
    // SURVEY.md §8 probe: C_R ~ 0.25-0.28 angles*N and DC(R^T R) ~ 0.95 angles*N
    CHECK(scale > 0.15 * A * n && scale < 0.4 * A * n, "calibrate_scale magnitude");
    CHECK(dc > 0.5 * A * n && dc < 1.5 * A * n, "dc response magnitude");
    SpectralMask meas = measurement_mask(geom, dc, 8, 0);
    CHECK(std::abs(meas.h[0].real() - dc) < 1e-9 * dc &&
              std::abs(meas.h[1].real() - scale) < 1e-9 * scale,
          "measurement_mask = radon_mask(n, scale, dc)");
    auto truth = randn(geom.domain_size(), 11);
    std::vector<double> sino(geom.range_size());
    geom.forward(truth, sino);
    ModelParams p;
    p.alpha = p.beta = 0.1;
    p.lambda = 0.01;
    SplitProblem prob = assemble_problem(sino, geom, p);
    SolverConfig cfg;
    cfg.alpha = p.alpha;
    cfg.mask = metric_mask(meas, p);
    cfg.max_iters = 3;
    cfg.record_every = 1;
    cfg.gamma = 1e-3;  // far below alpha lambda_max(A^T A - C): the screen warns
    SolveResult small = ncs_solve(prob, cfg);
    CHECK(!small.record.warnings.empty(), "screen warns on a violated step condition");
    cfg.gamma = 10.0 * A * n;  // comfortably above
    SolveResult big = ncs_solve(prob, cfg);
    CHECK(big.record.warnings.empty() && big.record.rows.size() == 4, "no warning when it holds");
    // admm_cg_solve (solvers.cpp:435-440): CG x-update, record axis in CG steps
    SolverConfig acfg;
    acfg.alpha = 0.5;
    acfg.max_iters = 6;
    acfg.record_every = 3;
    SolveResult adm = admm_cg_solve(prob, acfg, 4);
    CHECK(adm.record.rows.size() == 3 && adm.record.rows.back().iter == 24 &&
              std::isfinite(adm.objective),
          "admm_cg_solve runs, iterations counted in CG steps");
    bool rejected = false;
    try {
      admm_cg_solve(prob, cfg, 4);  // cfg has a mask
    } catch (const std::invalid_argument&) {
      rejected = true;
    }
    CHECK(rejected, "admm_cg_solve rejects a mask");
    write_record_csv("/tmp/ncsg_record_test.csv", big.record);
    std::ifstream in("/tmp/ncsg_record_test.csv");
    std::string header, first;
    std::getline(in, header);
    std::getline(in, first);
    CHECK(header == "iter,objective,rel_subopt,seminorm_step,wall_ms" && first.rfind("0,", 0) == 0,
          "write_record_csv format (io.cpp:203-215)");
  }
  // fan beam through SparseMap (fanbeam.cpp, sparse.cpp) and PET-TV (pipeline.cpp:84-89)
  {
    int n = 32;
    FanBeamGeometry fg = FanBeamGeometry::defaults(n, 24, 45);
    SparseMap A = build_fanbeam(n, fg);
    CHECK(A.nnz() > 0 && A.range_size() == 24u * 45u, "build_fanbeam SparseMap");
    auto x = randn(A.domain_size(), 21), u = randn(A.range_size(), 22);
    std::vector<double> ax(A.range_size()), atu(A.domain_size());
    A.forward(x, ax);
    A.adjoint(u, atu);
    double l = std::inner_product(ax.begin(), ax.end(), u.begin(), 0.0);
    double rr = std::inner_product(x.begin(), x.end(), atu.begin(), 0.0);
    CHECK(std::abs(l - rr) / std::max(1.0, std::abs(l)) <= 1e-5, "SparseMap adjoint probe");
    ModelParams p;
    p.alpha = p.beta = 0.1;
    p.lambda = 0.01;
    std::vector<double> truth(A.domain_size(), 0.0);
    for (int i = 8; i < 24; ++i)
      for (int j = 8; j < 24; ++j) truth[i * n + j] = 1.0;
    std::vector<double> sino(A.range_size());
    A.forward(truth, sino);
    SplitProblem prob = assemble_problem(sino, A, p);
    SolverConfig cfg;
    cfg.alpha = p.alpha;
    cfg.mask = metric_mask(measurement_mask(A, 0.0, 4, 0), p);
    cfg.gamma = 5.0 * 24 * n;
    cfg.max_iters = 20;
    cfg.record_every = 10;
    SolveResult r = ncs_solve(prob, cfg);
    CHECK(r.record.rows.size() == 3 && r.record.rows.back().objective < r.record.rows[0].objective,
          "fan-beam NCS solve decreases the objective");
    ModelParams pp = default_model_params("pet");
    pp.lambda = 0.01;
    RadonMap geom(n, 24, default_detector_count(n));
    std::vector<double> counts(geom.range_size());
    geom.forward(truth, counts);
    for (auto& c : counts) c = std::round(std::max(0.0, c) * 5.0);
    SplitProblem pet = assemble_problem(counts, geom, pp);
    SolverConfig pc;
    pc.alpha = pp.alpha;
    pc.gamma = 50.0;
    pc.max_iters = 10;
    pc.record_every = 5;
    pc.check_step_condition = false;
    SolveResult pr = pdhg_solve(pet, pc);
    // x0 = 0 gives y = 0 against positive counts: the Poisson objective is +inf
    // (PoissonConj::objective, prox.cpp:62-74), as in the reference
    CHECK(pet.kind == NCSG_PET && pr.state.u.size() == pet.range_size() &&
              std::isinf(pr.record.rows[0].objective) && pr.record.rows.size() == 3,
          "PET-TV problem (PoissonConj) solves");
  }
  // The reference's generic problem API (solvers.hpp:17-78): CT-TV built
  // block by block exactly as assemble_problem does (pipeline.cpp:84-97),
  // the denoising SplitProblem of test_solvers.cpp:646-664, Scaled mode of a
  // mask-free ncs_solve, and the m_pinv_override / m_override hooks.
  {
    int n = 32, A = 24, D = default_detector_count(n);
    auto geom = std::make_shared<const RadonMap>(n, A, D);
    auto truth = randn(geom->domain_size(), 31);
    for (auto& v : truth) v = std::max(0.0, v);
    std::vector<double> sino(geom->range_size());
    geom->forward(truth, sino);
    ModelParams p;
    p.alpha = p.beta = 0.1;
    p.lambda = 0.01;
    p.positivity = true;
    std::vector<SplitBlock> blocks;
    blocks.push_back({1.0, geom, std::make_shared<QuadraticConj>(), sino});
    blocks.push_back({p.beta / p.alpha, std::make_shared<GradMap>(n),
                      std::make_shared<ScaledL1Conj>(p.lambda * p.alpha / p.beta), {}});
    blocks.push_back({1.0, std::make_shared<IdentityMap>(geom->domain_size()),
                      std::make_shared<NonnegConj>(), {}});
    SplitProblem by_blocks(n, blocks);
    SplitProblem assembled = assemble_problem(sino, *geom, p);
    CHECK(by_blocks.range_size() == assembled.range_size() &&
              by_blocks.range_size() == geom->range_size() + 2u * n * (n - 1) + n * n &&
              by_blocks.block_offset(2) == geom->range_size() + 2u * n * (n - 1),
          "SplitProblem(n, blocks) stacked layout");
    SolverConfig cfg;
    cfg.alpha = p.alpha;
    cfg.gamma = 400.0;
    cfg.mask = metric_mask(radon_mask(n, 100.0, 400.0), p);
    cfg.max_iters = 20;
    cfg.record_every = 10;
    cfg.check_step_condition = false;
    SolveResult r1 = ncs_solve(by_blocks, cfg), r2 = ncs_solve(assembled, cfg);
    CHECK(r1.state.x.v == r2.state.x.v && r1.state.u == r2.state.u &&
              r1.objective == r2.objective,
          "block-built CT-TV problem == assemble_problem (bitwise)");
    // host objective of the block list against the device record
    double f_host = by_blocks.objective(r1.state.x.v);
    std::printf("  objective host %.9g device %.9g\n", f_host, r1.objective);
    CHECK((std::isinf(f_host) && std::isinf(r1.objective)) ||
              std::abs(f_host - r1.objective) <= 1e-5 * std::abs(f_host),
          "SplitProblem::objective");
    // Scaled mode: ncs_solve without a mask is pdhg_solve (mode_from, solvers.cpp:75-79)
    SolverConfig sc = cfg;
    sc.mask.reset();
    sc.gamma = 50.0 * A * n;
    SolveResult s1 = ncs_solve(by_blocks, sc), s2 = pdhg_solve(by_blocks, sc);
    CHECK(s1.state.x.v == s2.state.x.v && s1.state.u == s2.state.u,
          "mask-free ncs_solve == pdhg_solve (bitwise)");
    // Override mode with circulant metrics equals Mask mode
    SpectralMask m(n);
    for (std::size_t i = 0; i < m.h.size(); ++i) m.h[i] = cfg.gamma + cfg.alpha * cfg.mask->h[i];
    SolverConfig oc = cfg;
    oc.mask.reset();
    oc.m_pinv_override = std::make_shared<CirculantMap>(pinv_mask(m, cfg.pinv_rel_tol));
    oc.m_override = std::make_shared<CirculantMap>(m);
    SolveResult o1 = ncs_solve(by_blocks, oc);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < o1.state.x.v.size(); ++i) {
      num += std::pow(o1.state.x.v[i] - r1.state.x.v[i], 2);
      den += std::pow(r1.state.x.v[i], 2);
    }
    bool rows_ok = o1.record.rows.size() == r1.record.rows.size();
    for (std::size_t i = 0; rows_ok && i < o1.record.rows.size(); ++i)
      rows_ok = std::abs(o1.record.rows[i].seminorm_step - r1.record.rows[i].seminorm_step) <=
                1e-4 * std::max(1.0, std::abs(r1.record.rows[i].seminorm_step));
    CHECK(std::sqrt(num / den) <= 1e-6 && rows_ok,
          "m_pinv_override / m_override (CirculantMap) == mask mode");
    SolverConfig oc2 = oc;
    oc2.m_override.reset();
    bool need = false;
    try {
      ncs_solve(by_blocks, oc2);
    } catch (const std::invalid_argument& e) {
      need = std::string(e.what()).find("m_override is required") != std::string::npos;
    }
    CHECK(need, "m_override required alongside m_pinv_override");
    bool explicit_rejected = false;
    SolverConfig oc3 = oc;
    oc3.m_pinv_override = std::make_shared<GradMap>(n);  // not a circulant
    try {
      ncs_solve(by_blocks, oc3);
    } catch (const std::invalid_argument&) {
      explicit_rejected = true;
    }
    CHECK(explicit_rejected, "non-circulant metric override rejected");
    bool unsupported = false;
    try {
      std::vector<SplitBlock> one;
      one.push_back({10.0, std::make_shared<IdentityMap>(16), std::make_shared<QuadraticConj>(),
                     randn(16, 98)});
      SplitProblem bad(4, std::move(one));
    } catch (const std::invalid_argument& e) {
      unsupported = std::string(e.what()).find("no GPU kernel") != std::string::npos;
    }
    CHECK(unsupported, "block list without a device kernel rejected");
    bool dom = false;
    try {
      std::vector<SplitBlock> wrong;
      wrong.push_back({1.0, std::make_shared<GradMap>(8), std::make_shared<QuadraticConj>(), {}});
      SplitProblem bad(4, std::move(wrong));
    } catch (const std::invalid_argument& e) {
      dom = std::string(e.what()) == "block domain does not match the image size";
    }
    CHECK(dom, "SplitProblem validation message (solvers.cpp:346-347)");
    // TV denoising as the SplitProblem of test_solvers.cpp:646-664 / make_tv
    int nd = 16;
    auto noisy = randn(nd * nd, 41);
    std::vector<SplitBlock> tv;
    tv.push_back({1.0, std::make_shared<IdentityMap>(nd * nd), std::make_shared<QuadraticConj>(),
                  noisy});
    tv.push_back({0.05 / 0.05, std::make_shared<GradMap>(nd), std::make_shared<ScaledL1Conj>(0.3),
                  {}});
    SplitProblem tvp(nd, std::move(tv));
    ModelParams dp;
    dp.alpha = dp.beta = 0.05;
    dp.lambda = 0.3;
    SplitProblem tvd = denoise_problem(noisy, nd, dp);
    SolverConfig tc;
    tc.alpha = 0.05;
    tc.gamma = 1.0;
    tc.mask = laplacian_mask_2d(nd);
    tc.max_iters = 30;
    tc.record_every = 10;
    SolveResult t1 = ncs_solve(tvp, tc), t2 = ncs_solve(tvd, tc);
    CHECK(tvp.kind == NCSG_DENOISE && t1.state.x.v == t2.state.x.v && t1.objective == t2.objective,
          "denoising SplitProblem by blocks == denoise_problem (bitwise)");
    // an initial state is taken and replayed stepwise (test_solvers.cpp:607-625)
    SolverState init = make_state(tvp);
    init.x.v = randn(init.x.v.size(), 96);
    init.u = randn(init.u.size(), 97);
    tc.max_iters = 5;
    SolveResult ri = ncs_solve(tvp, tc, nullptr, &init);
    SolverState manual = init;
    manual.iter = 0;
    for (int k = 0; k < 5; ++k) ncs_step(manual, tvp, tc);
    CHECK(ri.state.x.v == manual.x.v && ri.state.u == manual.u && ri.state.iter == 5,
          "solve from an initial state replays the stepwise path");
  }
  // multi-GPU from C++: cfg.comm of an in-process group of 4 ranks (one host
  // thread each), orbit shards with the slab exchange, against the
  // unsharded solve
  {
    int n = 64, A = 48, D = default_detector_count(n);
    RadonMap geom(n, A, D);
    auto truth = randn(geom.domain_size(), 51);
    for (auto& v : truth) v = std::max(0.0, v);
    std::vector<double> sino(geom.range_size());
    geom.forward(truth, sino);
    ModelParams p;
    p.alpha = p.beta = 0.1;
    p.lambda = 0.01;
    SplitProblem prob = assemble_problem(sino, geom, p);
    SolverConfig cfg;
    cfg.alpha = p.alpha;
    cfg.gamma = 2000.0;
    cfg.mask = metric_mask(radon_mask(n, 0.27 * A * n, dc_response(geom)), p);
    cfg.max_iters = 20;
    cfg.record_every = 10;
    cfg.check_step_condition = false;
    SolveResult ref = ncs_solve(prob, cfg);
    auto comms = Communicator::local_group(4);
    std::vector<SolveResult> res(4);
    std::vector<std::thread> th;
    for (int r = 0; r < 4; ++r)
      th.emplace_back([&, r] {
        SolverConfig c = cfg;
        c.comm = comms[r];
        c.exchange = NCSG_XCHG_P2P;
        res[r] = ncs_solve(prob, c);
      });
    for (auto& t : th) t.join();
    bool ok = true;
    for (int r = 0; r < 4; ++r) {
      double num = 0, den = 0;
      for (std::size_t i = 0; i < ref.state.x.v.size(); ++i) {
        num += std::pow(res[r].state.x.v[i] - ref.state.x.v[i], 2);
        den += std::pow(ref.state.x.v[i], 2);
      }
      ok = ok && std::sqrt(num / den) <= 1e-5 &&
           std::abs(res[r].objective - ref.objective) <= 1e-5 * std::abs(ref.objective);
    }
    CHECK(ok, "4-rank P2P slab-sharded ncs_solve (cfg.comm) == unsharded");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
