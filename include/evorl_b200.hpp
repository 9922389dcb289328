// evorl_b200.hpp -- header-only C++17 host mirror of the reference's API over
// the C ABI (evorl_b200.h): the names a C++ caller of the reference uses for
// this path (proj/include/evorl/{workflow,ec,rollout,checkpoint}.hpp), the
// reference's exception types, and RAII ownership of the device workflow.
// Link with -levorl_b200.
#pragma once

#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
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
  // Workflow::step with the EsState held by the caller (mean and the Adam
  // moments, updated in place): one C-ABI call, one synchronisation
  StepMetrics step_host(std::vector<double>& mean, std::vector<double>& m, std::vector<double>& v,
                        std::int64_t& t) {
    const std::size_t d = (std::size_t)dim();
    if (mean.size() != d || m.size() != d || v.size() != d)
      throw std::invalid_argument("step_host: size mismatch");
    evorl_step_metrics met{};
    check(evorl_es_step_host(h_.get(), mean.data(), m.data(), v.data(), t, mean.data(), m.data(), v.data(), &t,
                             &met));
    return {met.fitness_mean, met.fitness_max, met.fitness_min, met.sigma, met.update_skipped != 0};
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
  // WorkflowState::rng: the key of init() or of the loaded checkpoint
  RngKey rng() const {
    RngKey k;
    check(evorl_es_get_rng(h_.get(), &k.hi, &k.lo));
    return k;
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

// ------------------------------------------------------ metrics stream
// MetricsWriter (proj/include/evorl/metrics.hpp, proj/src/metrics.cpp:12-67):
// metrics.jsonl (one nlohmann::json dump() per line: keys sorted, no
// whitespace, doubles shortest round-trip placed as nlohmann's format_buffer
// does, non-finite -> null) and the timings sidecar.  paper_2501_15129_b200/
// learn.py writes the same bytes.
namespace detail {
inline std::string json_double(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, std::fabs(x), std::chars_format::scientific);
  const std::string sci(buf, r.ptr);  // d[.ddd]e[+-]XX, shortest round-trip
  const std::size_t epos = sci.find('e');
  std::string ds = sci.substr(0, epos);
  if (ds.size() > 1) ds.erase(1, 1);  // drop the '.'
  while (ds.size() > 1 && ds.back() == '0') ds.pop_back();
  const int k = (int)ds.size(), n = std::atoi(sci.c_str() + epos + 1) + 1;
  std::string out = x < 0 ? "-" : "";
  if (k <= n && n <= 15) return out + ds + std::string((std::size_t)(n - k), '0') + ".0";
  if (0 < n && n <= 15) return out + ds.substr(0, (std::size_t)n) + "." + ds.substr((std::size_t)n);
  if (-4 < n && n <= 0) return out + "0." + std::string((std::size_t)-n, '0') + ds;
  const int e = n - 1;
  out += k == 1 ? ds : ds.substr(0, 1) + "." + ds.substr(1);
  char eb[16];
  std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
  return out + eb;
}
inline std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char u[16];
          std::snprintf(u, sizeof u, "\\u%04x", c);
          o += u;
        } else {
          o += (char)c;
        }
    }
  }
  return o + "\"";
}
// a flat JSON object: key -> already-serialised value, emitted in std::map order
inline std::string json_object(const std::map<std::string, std::string>& kv) {
  std::string o = "{";
  for (const auto& [k, v] : kv) {
    if (o.size() > 1) o += ',';
    o += json_string(k) + ":" + v;
  }
  return o + "}";
}
}  // namespace detail

class MetricsWriter {
 public:
  MetricsWriter(const std::string& metrics_path, const std::string& timings_path)
      : metrics_(metrics_path, std::ios::trunc), timings_(timings_path, std::ios::trunc) {
    if (!metrics_) throw std::runtime_error("cannot open metrics file: " + metrics_path);
    if (!timings_) throw std::runtime_error("cannot open timings file: " + timings_path);
  }
  void write_header(const std::string& workflow_id, const std::map<std::string, std::string>& config) {
    std::map<std::string, std::string> conf;
    for (const auto& [k, v] : config) conf[k] = detail::json_string(v);
    metrics_ << detail::json_object({{"type", "\"header\""},
                                     {"workflow", detail::json_string(workflow_id)},
                                     {"config", detail::json_object(conf)}})
             << '\n';
    flush();
  }
  void write_step(std::int64_t iteration, std::int64_t env_steps, std::int64_t episodes,
                  std::int64_t rl_updates, const std::vector<std::pair<std::string, double>>& scalars) {
    auto rec = base("step", iteration, env_steps, episodes, rl_updates);
    for (const auto& [k, v] : scalars) rec[k] = detail::json_double(v);
    metrics_ << detail::json_object(rec) << '\n';
  }
  void write_eval(std::int64_t iteration, std::int64_t env_steps, std::int64_t episodes,
                  std::int64_t rl_updates, double mean_return, double return_std, int eval_episodes) {
    auto rec = base("eval", iteration, env_steps, episodes, rl_updates);
    rec["eval/episode_return_mean"] = detail::json_double(mean_return);
    rec["eval/episode_return_std"] = detail::json_double(return_std);
    rec["eval/episodes"] = std::to_string(eval_episodes);
    metrics_ << detail::json_object(rec) << '\n';
    flush();
  }
  void write_timing(std::int64_t iteration, double wall_ms) { timings_ << iteration << '\t' << wall_ms << '\n'; }
  void flush() {
    metrics_.flush();
    timings_.flush();
  }

 private:
  static std::map<std::string, std::string> base(const char* type, std::int64_t it, std::int64_t steps,
                                                 std::int64_t eps, std::int64_t rl) {
    return {{"type", detail::json_string(type)}, {"iteration", std::to_string(it)},
            {"env_steps", std::to_string(steps)}, {"episodes", std::to_string(eps)},
            {"rl_updates", std::to_string(rl)}};
  }
  std::ofstream metrics_, timings_;
};

// Budget / LearnOptions / learn (proj/include/evorl/workflow.hpp:74-98,
// proj/src/workflow.cpp:46-68) over the device workflow.  Eval keys derive
// from the handle's own WorkflowState::rng (fold_in(fold_in(rng, 1), it),
// proj/include/evorl/workflow.hpp:42), so a resumed workflow evaluates like the
// reference; a caller key that differs from the state's throws invalid_argument.
struct Budget {
  std::int64_t iterations = 0, episodes = 0, env_steps = 0;  // 0 = off
  bool reached(std::int64_t it, std::int64_t steps, std::int64_t eps) const {
    return (iterations > 0 && it >= iterations) || (episodes > 0 && eps >= episodes) ||
           (env_steps > 0 && steps >= env_steps);
  }
};
struct LearnOptions {
  Budget budget;
  int eval_interval = 10;
  int eval_episodes = 128;
  int checkpoint_interval = 0;
  std::string checkpoint_path;
};
inline std::vector<std::pair<std::string, double>> step_scalars(const StepMetrics& m) {
  // EsWorkflow::step's StepMetrics (proj/src/workflow_es.cpp:140-169)
  return {{"es/sigma", m.sigma}, {"fitness/mean", m.fitness_mean}, {"fitness/max", m.fitness_max},
          {"fitness/min", m.fitness_min}, {"es/update_skipped", m.update_skipped ? 1.0 : 0.0}};
}
inline void learn(EsWorkflow& wf, const LearnOptions& opt, MetricsWriter& metrics) {
  using clock = std::chrono::steady_clock;
  const RngKey rng = wf.rng();
  std::int64_t it = 0, steps = 0, eps = 0;
  for (wf.counters(&it, &steps, &eps); !opt.budget.reached(it, steps, eps);) {
    const auto t0 = clock::now();
    const StepMetrics sm = wf.step();
    const double ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
    wf.counters(&it, &steps, &eps);
    metrics.write_step(it, steps, eps, 0, step_scalars(sm));
    metrics.write_timing(it, ms);
    if (opt.eval_interval > 0 && it % opt.eval_interval == 0) {
      const EvalReport er = wf.evaluate(opt.eval_episodes, fold_in(fold_in(rng, 1), (std::uint64_t)it));
      metrics.write_eval(it, steps, eps, 0, er.mean_return, er.return_std, er.episodes);
    }
    if (opt.checkpoint_interval > 0 && !opt.checkpoint_path.empty() && it % opt.checkpoint_interval == 0)
      wf.save(opt.checkpoint_path);
  }
  if (!opt.checkpoint_path.empty()) wf.save(opt.checkpoint_path);
  metrics.flush();
}
inline void learn(EsWorkflow& wf, RngKey rng, const LearnOptions& opt, MetricsWriter& metrics) {
  const RngKey st = wf.rng();
  if (rng.hi != st.hi || rng.lo != st.lo)
    throw std::invalid_argument("learn(): rng is not the workflow state's key (eval keys derive from WorkflowState::rng)");
  learn(wf, opt, metrics);
}

}  // namespace evorl_b200
