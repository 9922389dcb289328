// env.cuh -- classic-control dynamics on the device, fp64, evaluated in the
// reference's operation order with no FMA contraction (dmul/dadd/...).
// Restates proj/src/env.cpp:28-155 (CartPole Euler dt=0.02, Pendulum
// semi-implicit Euler dt=0.05, auto-reset from the episode's own key).
#pragma once

#include "common.cuh"

namespace evorl_b200 {

enum : int { ENV_CARTPOLE = 0, ENV_PENDULUM = 1 };

struct EnvDesc {
  int id;
  int obs_dim;
  int act_dim;
  int discrete;
  int num_actions;
  int max_episode_steps;
  int fixed_horizon;
  double act_low, act_high;
};

struct LaneEnv {
  double p0, p1, p2, p3;  // CartPole: x, xdot, th, thdot; Pendulum: th, thdot
  int step_count;
  DKey rng;  // the episode's auto-reset key (proj/include/evorl/env.hpp:41-45)
};

#define EVB_PI 3.141592653589793

// fmod(x, y) for finite y > 0, bit-identical to the library fmod (which is
// exact): for |x| < 2^40 y the truncated quotient estimate from the rounded
// reciprocal is off by at most one, the remainder x - n*y of the right n is
// representable so one fma yields it exactly, and a wrong n shows up as a
// remainder outside [0, y) (rounding is monotone) and is corrected once.
EVB_DEV double fmod_exact(double x, double y, double inv_y) {
  const double ax = fabs(x);
  if (!(ax < 1099511627776.0 * y)) return fmod(x, y);  // huge or non-finite: library path
  double n = trunc(ax * inv_y);
  double r = fma(-n, y, ax);
  if (r < 0.0) {
    n -= 1.0;
    r = fma(-n, y, ax);
  } else if (r >= y) {
    n += 1.0;
    r = fma(-n, y, ax);
  }
  return copysign(r, x);
}

// proj/src/env.cpp:28-32: fmod is exact; the adds are single rounded ops.
EVB_DEV double wrap_angle(double th) {
  double w = fmod_exact(dadd(th, EVB_PI), 6.283185307179586, 1.0 / 6.283185307179586);
  if (w <= 0.0) w = dadd(w, 6.283185307179586);
  return dsub(w, EVB_PI);
}

EVB_DEV double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }

// proj/src/env.cpp:87-97
EVB_DEV void observe(const EnvDesc& e, const LaneEnv& s, double* obs) {
  if (e.id == ENV_CARTPOLE) {
    obs[0] = s.p0;
    obs[1] = s.p1;
    obs[2] = s.p2;
    obs[3] = s.p3;
  } else {
    double sn, cs;
    sincos(s.p0, &sn, &cs);
    obs[0] = cs;
    obs[1] = sn;
    obs[2] = s.p1;
    obs[3] = 0.0;
  }
}

// proj/src/env.cpp:99-111: initial conditions from RandomStream(fold_in(key, 0)),
// state.rng = fold_in(key, 1).
EVB_DEV void env_reset(const EnvDesc& e, DKey key, LaneEnv& s) {
  const DKey sk = fold_in(key, 0);
  uint64_t w0, w1;
  threefry2x64(sk.hi, sk.lo, 1, 0, w0, w1);
  if (e.id == ENV_CARTPOLE) {
    uint64_t w2, w3;
    threefry2x64(sk.hi, sk.lo, 1, 1, w2, w3);
    s.p0 = uniform_range(-0.05, 0.05, word_to_uniform(w0));
    s.p1 = uniform_range(-0.05, 0.05, word_to_uniform(w1));
    s.p2 = uniform_range(-0.05, 0.05, word_to_uniform(w2));
    s.p3 = uniform_range(-0.05, 0.05, word_to_uniform(w3));
  } else {
    s.p0 = uniform_range(-EVB_PI, EVB_PI, word_to_uniform(w0));
    s.p1 = uniform_range(-1.0, 1.0, word_to_uniform(w1));
    s.p2 = 0.0;
    s.p3 = 0.0;
  }
  s.step_count = 0;
  s.rng = fold_in(key, 1);
}

// One env_step (proj/src/env.cpp:113-155).  Returns 0 or a FAULT_* kind.
// sin_th (optional): sin of the current angle, already computed by observe()
// for this state -- the reference evaluates std::sin(th) twice with the same
// argument (proj/src/env.cpp:94 and :48), so reusing it is exact.
// pendulum_reward_pre: the action-independent part of the Pendulum reward,
// w*w + (0.1*thdot)*thdot with w = wrap_angle(th) (proj/src/env.cpp:139-141),
// so a caller can evaluate it off the action's critical path; env_step then
// adds (0.001*u)*u in the reference's order (bit-identical).
EVB_DEV double pendulum_reward_pre(const LaneEnv& s) {
  const double w = wrap_angle(s.p0);
  return dadd(dmul(w, w), dmul(dmul(0.1, s.p1), s.p1));
}

EVB_DEV uint32_t env_step(const EnvDesc& e, LaneEnv& s, double action, double& reward,
                          bool& terminated, bool& truncated, const double* sin_th = nullptr,
                          const double* reward_pre = nullptr) {
  const bool cart = e.id == ENV_CARTPOLE;
  if (!isfinite(s.p0) || !isfinite(s.p1) || (cart && (!isfinite(s.p2) || !isfinite(s.p3))))
    return FAULT_ENV_STATE;
  if (!isfinite(action)) return FAULT_ENV_ACTION;
  terminated = false;
  if (cart) {
    const double force = action > 0.5 ? 10.0 : -10.0;
    const double x = s.p0, xdot = s.p1, th = s.p2, thdot = s.p3;
    double sinth, costh;
    sincos(th, &sinth, &costh);
    // temp = (force + ((0.05*thdot)*thdot)*sinth) / 1.1
    const double temp = ddiv(dadd(force, dmul(dmul(dmul(0.05, thdot), thdot), sinth)), 1.1);
    // thacc = (9.8*sinth - costh*temp) / (0.5*(4/3 - ((0.1*costh)*costh)/1.1))
    const double num = dsub(dmul(9.8, sinth), dmul(costh, temp));
    const double den =
        dmul(0.5, dsub(4.0 / 3.0, ddiv(dmul(dmul(0.1, costh), costh), 1.1)));
    const double thacc = ddiv(num, den);
    // xacc = temp - ((0.05*thacc)*costh)/1.1
    const double xacc = dsub(temp, ddiv(dmul(dmul(0.05, thacc), costh), 1.1));
    s.p0 = dadd(x, dmul(0.02, xdot));
    s.p1 = dadd(xdot, dmul(0.02, xacc));
    s.p2 = dadd(th, dmul(0.02, thdot));
    s.p3 = dadd(thdot, dmul(0.02, thacc));
    reward = 1.0;
    if (!e.fixed_horizon)
      terminated = fabs(s.p0) > 2.4 || fabs(s.p2) > 0.20943951023931953;  // 12*pi/180
  } else {
    const double u = clampd(action, -2.0, 2.0);
    const double th = s.p0, thdot = s.p1;
    // -((w*w + (0.1*thdot)*thdot) + (0.001*u)*u)
    const double pre = reward_pre ? *reward_pre : pendulum_reward_pre(s);
    reward = -dadd(pre, dmul(dmul(0.001, u), u));
    // pendulum_physics (proj/src/env.cpp:46-51), 1.5*kPenG = 15 exactly
    const double sn = sin_th ? *sin_th : sin(th);
    double td = dadd(thdot, dmul(dadd(dmul(15.0, sn), dmul(3.0, u)), 0.05));
    td = clampd(td, -8.0, 8.0);
    s.p0 = dadd(th, dmul(td, 0.05));
    s.p1 = td;
  }
  s.step_count += 1;
  truncated = s.step_count >= e.max_episode_steps && !terminated;
  if (!isfinite(s.p0) || !isfinite(s.p1) || (cart && (!isfinite(s.p2) || !isfinite(s.p3))))
    return FAULT_ENV_SUCCESSOR;
  return 0;
}

}  // namespace evorl_b200
