// es_generation.cpp -- a C++ host running EsWorkflow generations on the B200
// through evorl_b200.hpp, the way the reference's learn() loop drives its
// Workflow (proj/src/workflow.cpp:46-68): init, step, periodic evaluate,
// checkpoint.  Prints one line per generation (values in %a for exact
// comparison) and the final counters.
//
//   es_generation [algo] [pop] [gens] [hidden0] [hidden1] [episodes] [precision] [checkpoint]
//   es_generation learn <out_dir>      learn() + metrics.jsonl / timings.log / checkpoint.bin
//   es_generation cma-sphere           the reference's CMA offset-sphere test via CmaEs
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "evorl_b200.hpp"

int main(int argc, char** argv) {
  namespace eb = evorl_b200;
  const char* algo = argc > 1 ? argv[1] : "openes";
  if (!std::strcmp(algo, "learn") && argc > 2) {  // learn() + metrics stream (proj/src/workflow.cpp:46-68)
    try {
      evorl_es_config c = eb::default_config();
      c.env_id = EVORL_ENV_PENDULUM;
      c.fixed_horizon = 1;
      c.max_episode_steps = 60;
      c.pop = 32;
      c.n_hidden = 2;
      c.hidden[0] = c.hidden[1] = 16;
      c.vbn_samples = 300;
      const std::string dir = argv[2];
      const eb::RngKey root = eb::key_from_seed(3);
      eb::EsWorkflow wf(c);
      wf.init(root);
      eb::MetricsWriter mw(dir + "/metrics.jsonl", dir + "/timings.log");
      mw.write_header("es", {{"workflow", "es"}, {"seed", "3"}, {"ec.pop", "32"}});
      eb::LearnOptions lo;
      lo.budget.iterations = 5;
      lo.eval_interval = 2;
      lo.eval_episodes = 8;
      lo.checkpoint_path = dir + "/checkpoint.bin";
      eb::learn(wf, root, lo, mw);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 2;
    }
    return 0;
  }
  if (!std::strcmp(algo, "cma-sphere")) {  // proj/tests/test_ec.cpp:282-297 through the free functions
    try {
      const double target[8] = {0.7, -0.3, 0.5, 0.1, -0.8, 0.25, -0.4, 0.6};
      eb::CmaEs cma(8, 16, 8, 0.3);
      for (int g = 0; g < 200; ++g) {
        const std::vector<double> cand = cma.ask(eb::fold_in(eb::key_from_seed(84), (std::uint64_t)g));
        std::vector<double> fit(16);
        for (int i = 0; i < 16; ++i) {
          double s2 = 0;
          for (int j = 0; j < 8; ++j) s2 += (cand[i * 8 + j] - target[j]) * (cand[i * 8 + j] - target[j]);
          fit[i] = -s2;
        }
        cma.tell(cand, fit);
      }
      const std::vector<double> m = cma.mean();
      double dist = 0;
      for (int j = 0; j < 8; ++j) dist += (m[j] - target[j]) * (m[j] - target[j]);
      std::printf("cma-sphere distance %a sigma %a\n", std::sqrt(dist), cma.sigma());
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 2;
    }
    return 0;
  }
  evorl_es_config cfg = eb::default_config();
  cfg.algo = !std::strcmp(algo, "ars") ? EVORL_ALGO_ARS : !std::strcmp(algo, "cmaes") ? EVORL_ALGO_CMAES
                                                                                      : EVORL_ALGO_OPENES;
  cfg.env_id = EVORL_ENV_PENDULUM;
  cfg.fixed_horizon = 1;
  cfg.max_episode_steps = 100;
  cfg.pop = argc > 2 ? std::atoi(argv[2]) : 64;
  const int gens = argc > 3 ? std::atoi(argv[3]) : 3;
  cfg.n_hidden = 2;
  cfg.hidden[0] = argc > 4 ? std::atoi(argv[4]) : 32;
  cfg.hidden[1] = argc > 5 ? std::atoi(argv[5]) : 32;
  cfg.fitness_episodes = argc > 6 ? std::atoi(argv[6]) : 1;
  const std::string prec = argc > 7 ? argv[7] : "f64";
  cfg.precision = prec == "tc" ? EVORL_PREC_TC : prec == "f32" ? EVORL_PREC_F32 : EVORL_PREC_F64;
  cfg.vbn_samples = 500;
  try {
    eb::EsWorkflow wf(cfg);
    wf.init({0x1234, 0x5678});
    for (int g = 0; g < gens; ++g) {
      const eb::StepMetrics m = wf.step();
      std::printf("gen %d fitness_mean %a fitness_max %a sigma %a skipped %d\n", g, m.fitness_mean,
                  m.fitness_max, m.sigma, m.update_skipped ? 1 : 0);
    }
    const eb::EvalReport ev = wf.evaluate(16, {7, 8});
    std::printf("eval mean %a std %a\n", ev.mean_return, ev.return_std);
    std::int64_t it = 0, steps = 0, eps = 0;
    wf.counters(&it, &steps, &eps);
    std::printf("counters %lld %lld %lld\n", (long long)it, (long long)steps, (long long)eps);
    if (argc > 8) wf.save(argv[8]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
