// evorl_b200.hpp -- header-only C++17 host mirror of the reference's API over
// the C ABI (evorl_b200.h): the names a C++ caller of the reference uses for
// this path (proj/include/evorl/{workflow,ec,rollout,checkpoint}.hpp), the
// reference's exception types, and RAII ownership of the device workflow.
// Link with -levorl_b200.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "evorl_b200.h"

namespace evorl_b200 {

// ----------------------------------------------------------------- errors
// The status codes map 1:1 onto the reference's exception types
// (proj/src/ec.cpp invalid_argument / length_error, proj/include/evorl/
// env.hpp:19-21 EnvFault, net.hpp:19-21 NetFault, config.hpp:11-13
// ConfigError, checkpoint.hpp:14-16 CheckpointError); what() is the
// reference's message text.
struct EnvFault : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NetFault : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CheckpointError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {  // CUDA / no device (there is no CPU fallback)
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {  // a valid reference input the device path refuses
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == EVORL_OK) return;
  const std::string msg = evorl_last_error();
  switch (rc) {
    case EVORL_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case EVORL_E_LENGTH: throw std::length_error(msg);
    case EVORL_E_ENV_FAULT: throw EnvFault(msg);
    case EVORL_E_NET_FAULT: throw NetFault(msg);
    case EVORL_E_CONFIG: throw ConfigError(msg);
    case EVORL_E_CHECKPOINT: throw CheckpointError(msg);
    case EVORL_E_UNSUPPORTED: throw Unsupported(msg);
    default: throw DeviceError(msg);
  }
}

// RngKey (proj/include/evorl/rng.hpp)
struct RngKey {
  std::uint64_t hi = 0, lo = 0;
};

// key_from_seed / fold_in (proj/src/rng.cpp:36-46) over evorl_threefry2x64
inline RngKey fold_in(RngKey key, std::uint64_t index) {
  const std::uint64_t k[2] = {key.hi, key.lo}, c[2] = {0, index};
  std::uint64_t o[2];
  check(evorl_threefry2x64(k, c, o, 1));
  return {o[0], o[1]};
}
inline RngKey key_from_seed(std::uint64_t seed) {
  return fold_in({0x9E3779B97F4A7C15ull, 0xBB67AE8584CAA73Bull}, seed);
}

// StepMetrics / EvalReport (proj/include/evorl/workflow.hpp)
struct StepMetrics {
  double fitness_mean = 0, fitness_max = 0, fitness_min = 0, sigma = 0;
  bool update_skipped = false;
};
struct EvalReport {
  double mean_return = 0, return_std = 0;
  int episodes = 0;
};

inline evorl_es_config default_config() {
  evorl_es_config c;
  evorl_es_default_config(&c);
  return c;
}

// --------------------------------------------------------------- workflow
// EsWorkflow (proj/src/workflow_es.cpp): the generation step on the device,
// state resident in HBM.  init / step / evaluate / save / load as the
// reference's Workflow virtuals (proj/include/evorl/workflow.hpp:48-70).
class EsWorkflow {
 public:
  explicit EsWorkflow(const evorl_es_config& cfg) {
    evorl_es* h = nullptr;
    check(evorl_es_create(&cfg, &h));
    h_.reset(h);
  }
  std::int64_t dim() const { return evorl_es_dim(h_.get()); }

  EsWorkflow& init(RngKey key) {
    check(evorl_es_init(h_.get(), key.hi, key.lo));
    return *this;
  }
  StepMetrics step() {
    evorl_step_metrics m{};
    check(evorl_es_step(h_.get(), &m));
    return {m.fitness_mean, m.fitness_max, m.fitness_min, m.sigma, m.update_skipped != 0};
  }
  EvalReport evaluate(int episodes, RngKey key) {
    EvalReport r;
    check(evorl_es_evaluate(h_.get(), episodes, key.hi, key.lo, &r.mean_return, &r.return_std));
    r.episodes = episodes;
    return r;
  }
  // checkpoint_save / checkpoint_load of an "es" workflow (EVORL1 files)
  void save(const std::string& path) { check(evorl_es_save(h_.get(), path.c_str())); }
  EsWorkflow& load(const std::string& path) {
    check(evorl_es_load(h_.get(), path.c_str()));
    return *this;
  }

  // state access (EsState, proj/src/workflow_es.cpp:15-20)
  std::vector<double> mean() {
    std::vector<double> v((std::size_t)dim());
    check(evorl_es_get_mean(h_.get(), v.data()));
    return v;
  }
  void set_mean(const std::vector<double>& v) {
    if ((std::int64_t)v.size() != dim()) throw std::invalid_argument("set_mean: size mismatch");
    check(evorl_es_set_mean(h_.get(), v.data()));
  }
  std::vector<double> fitness(int pop) {
    std::vector<double> f((std::size_t)pop);
    check(evorl_es_get_fitness(h_.get(), f.data()));
    return f;
  }
  void counters(std::int64_t* iteration, std::int64_t* env_steps, std::int64_t* episodes) const {
    check(evorl_es_counters(h_.get(), iteration, env_steps, episodes));
  }
  evorl_es* handle() { return h_.get(); }

 private:
  struct Del {
    void operator()(evorl_es* h) const { evorl_es_destroy(h); }
  };
  std::unique_ptr<evorl_es, Del> h_;
};

// ------------------------------------------------------------- CMA-ES
// CmaState::init / cmaes_ask / cmaes_tell (proj/src/ec.cpp:191-288) on a
// device state of dimension d; the caller evaluates the candidates.
class CmaEs {
 public:
  CmaEs(std::int64_t d, int pop, int elites, double sigma0, int max_dim = 4096, int eig_every = 1)
      : d_(d), pop_(pop) {
    evorl_es* h = nullptr;
    check(evorl_cma_create(d, pop, elites, sigma0, max_dim, eig_every, &h));
    h_.reset(h);
  }
  // pop x d row-major candidates
  std::vector<double> ask(RngKey key) {
    std::vector<double> c((std::size_t)(pop_ * d_));
    check(evorl_cma_ask(h_.get(), key.hi, key.lo, c.data()));
    return c;
  }
  void tell(const std::vector<double>& candidates, const std::vector<double>& fitness) {
    if ((std::int64_t)candidates.size() != pop_ * d_ || (int)fitness.size() != pop_)
      throw std::invalid_argument("cmaes_tell: candidates / fitness size mismatch");
    check(evorl_cma_tell(h_.get(), candidates.data(), fitness.data()));
  }
  std::vector<double> mean() {
    std::vector<double> v((std::size_t)d_);
    check(evorl_es_get_mean(h_.get(), v.data()));
    return v;
  }
  void set_mean(const std::vector<double>& v) {
    if ((std::int64_t)v.size() != d_) throw std::invalid_argument("set_mean: size mismatch");
    check(evorl_es_set_mean(h_.get(), v.data()));
  }
  double sigma() {
    double s = 0;
    check(evorl_es_cma_get(h_.get(), nullptr, nullptr, nullptr, nullptr, nullptr, &s, nullptr, nullptr));
    return s;
  }

 private:
  struct Del {
    void operator()(evorl_es* h) const { evorl_es_destroy(h); }
  };
  std::int64_t d_;
  int pop_;
  std::unique_ptr<evorl_es, Del> h_;
};

// ------------------------------------------------------ free functions
// centered_ranks / rank_desc (proj/src/ec.cpp:14-46)
inline std::vector<double> centered_ranks(const std::vector<double>& f) {
  std::vector<double> out(f.size());
  check(evorl_centered_ranks(f.data(), (std::int64_t)f.size(), out.data()));
  return out;
}
inline std::vector<std::int32_t> rank_desc(const std::vector<double>& f) {
  std::vector<std::int32_t> out(f.size());
  check(evorl_rank_desc(f.data(), (std::int64_t)f.size(), out.data()));
  return out;
}
// gaussian_matrix (proj/src/ec.cpp:22-28), row-major rows x cols
inline std::vector<double> gaussian_matrix(RngKey key, std::int64_t rows, std::int64_t cols) {
  std::vector<double> out((std::size_t)(rows * cols));
  check(evorl_gaussian_matrix(key.hi, key.lo, rows, cols, out.data()));
  return out;
}

// batched_rollout (proj/src/rollout.cpp:176-214), deterministic policy,
// Episodes mode: params m x d row-major; returns m x count episode returns
// (lane-major order) and per-agent step counts.
struct RolloutResult {
  std::vector<double> returns;     // m x count
  std::vector<std::int64_t> steps; // m
};
inline RolloutResult batched_rollout(const evorl_env_desc& env, const evorl_mlp_desc& net,
                                     const evorl_obs_norm* norm, const std::vector<double>& params,
                                     int m, int envs_per_agent, int count, RngKey key,
                                     int precision = EVORL_PREC_F64) {
  RolloutResult r;
  r.returns.resize((std::size_t)m * count);
  r.steps.resize((std::size_t)m);
  check(evorl_batched_rollout(&env, &net, norm, params.data(), m, envs_per_agent, count, key.hi, key.lo,
                              precision, r.returns.data(), r.steps.data(), nullptr));
  return r;
}

}  // namespace evorl_b200
