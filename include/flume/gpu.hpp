// flume/gpu.hpp -- C++ drop-in adapter for the reference engine (proj/include/flume).
//
// Header-only; include it next to the reference headers and link
// libflume_b200.so.  It re-exposes the reference's hot-path signatures for
// D = 3 with a device workspace in place of MpmWorkspace<3>:
//
//   reference (proj/include/flume)                      this header
//   mpm_substep(scene, state, action, MpmWorkspace&)    gpu::mpm_substep(scene, state, action, gpu::Workspace&)
//     mpm.hpp:455-473
//   rollout_loss(scene, state0, actions, loss, ...)     gpu::rollout_loss(scene, state0, actions, loss_spec, ws, ...)
//     grad.hpp:15-41
//   grad_trajectory(scene, state0, actions, loss, ...)  gpu::grad_trajectory(scene, state0, actions, loss_spec, ws, ...)
//     grad.hpp:61-134
//   adjoint_substep(scene, rec, adj, action_bar, ws)    gpu::adjoint_substep(scene, rec, adj, action_bar, ws)
//     adjoint.hpp:476-548
//   grad_check(scene, state0, actions, loss, stride, eps) gpu::grad_check(scene, state0, actions, loss_spec, ws, ...)
//     grad.hpp:190-225
//
// The loss is passed as the scene's loss JSON (World::loss_spec, the input of
// LossEvaluator, losses.hpp:311) because LossEvaluator keeps its terms private;
// target_point, hold_initial, chamfer, mixing_spread (with the attraction term)
// and composite specs are evaluated on the device.
// Errors rethrow the reference exception types (core.hpp:18-48).
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <string>
#include <vector>

#include "flume/grad.hpp"
#include "flume_b200.h"

namespace flume {
namespace gpu {

inline void check(flume_ctx* ctx, int rc) {
    if (rc == FLUME_OK) return;
    flume_error_info info{};
    flume_last_error(ctx, &info);
    std::string msg(info.message);
    switch (rc) {
        case FLUME_E_SCENE: throw SceneError(msg);
        case FLUME_E_DEGENERATE: throw DegenerateDeformation(msg, info.particle_id);
        case FLUME_E_RIGIDITY: throw RigidityError(msg, info.body_id);
        case FLUME_E_ADJOINT: throw AdjointError(msg, info.substep);
        case FLUME_E_SOLVER: throw SolverError(msg);
        default: throw EngineError(msg);
    }
}

// Device context for one Scene<3> (the MpmWorkspace<3> analogue).  The scene's
// per-particle constants (material, body, mass, volume0, activation substep)
// and effector shapes are taken from the state given at construction.
// one rank of an x-slab group spanning processes (one per GPU, NCCL); uid from
// flume_dist_unique_id() on rank 0, shared by the launcher.  Every gpu:: call on
// such a workspace is collective over the ranks.
struct SlabRank {
    int rank = 0;
    int n_ranks = 1;
    const unsigned char* uid = nullptr;
};

// A replica context: `n` copies of the scene in one device context, every kernel launch
// covering all of them (flume_ctx_create_replicas; the CMA-ES population of
// optimize.hpp:383-418).  Use with rollout_loss_replicas.
struct Replicas {
    int n = 1;
};

class Workspace {
public:
    Workspace(const Scene<3>& scene, const SimState<3>& state, int device = 0, const SlabRank* slab = nullptr)
        : scene_(&scene) {
        build_desc(scene, state);
        if (slab && slab->n_ranks > 1)
            check(nullptr, flume_ctx_create_dist(&desc_, device, slab->rank, slab->n_ranks, slab->uid, &ctx_));
        else
            check(nullptr, flume_ctx_create(&desc_, device, &ctx_));
    }
    Workspace(const Scene<3>& scene, const SimState<3>& state, Replicas rep, int device = 0)
        : scene_(&scene), n_rep_(rep.n) {
        build_desc(scene, state);
        check(nullptr, flume_ctx_create_replicas(&desc_, rep.n, device, &ctx_));
    }
    ~Workspace() { flume_ctx_destroy(ctx_); }
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;

    flume_ctx* ctx() const { return ctx_; }
    const Scene<3>& scene() const { return *scene_; }
    int replicas() const { return n_rep_; }

private:
    void build_desc(const Scene<3>& scene, const SimState<3>& state) {
        const SimConfig<3>& c = scene.config;
        desc_.config.grid_resolution = c.grid_resolution;
        for (int a = 0; a < 3; a++) {
            desc_.config.domain[a] = c.domain_extent[a];
            desc_.config.gravity[a] = c.gravity[a];
        }
        desc_.config.dt_substep = c.dt_substep;
        desc_.config.substeps_per_step = c.substeps_per_step;
        desc_.config.boundary_width = c.boundary_width;
        desc_.config.contact_eps_cells = c.contact_eps_cells;
        desc_.config.cfl_fraction = c.cfl_fraction;
        desc_.config.mass_epsilon = c.mass_epsilon;
        desc_.config.hard_contact = c.hard_contact ? 1 : 0;
        for (const MaterialParams& m : scene.materials)
            mats_.push_back({int(m.kind), m.mu, m.lambda, m.rho, m.yield.theta_c, m.yield.theta_s, m.yield.sigma_y});
        for (const Effector<3>& e : state.effectors) {
            flume_effector_shape s{};
            s.shape_kind = int(e.sdf.shape.kind);
            s.radius = e.sdf.shape.radius;
            s.plane_offset = e.sdf.shape.plane_offset;
            s.half_height = e.sdf.shape.half_height;
            for (int a = 0; a < 3; a++) {
                s.half_extents[a] = e.sdf.shape.half_extents[a];
                s.seg_a[a] = e.sdf.shape.seg_a[a];
                s.seg_b[a] = e.sdf.shape.seg_b[a];
                s.plane_normal[a] = e.sdf.shape.plane_normal[a];
                s.shape_t[a] = e.sdf.pose.t[a];
            }
            for (int r = 0; r < 3; r++)
                for (int q = 0; q < 3; q++) s.shape_R[3 * r + q] = e.sdf.pose.R[r][q];
            s.friction_mu = e.friction_mu;
            for (int a = 0; a < 6; a++) s.action_mask[a] = e.action_mask[size_t(a)] ? 1 : 0;
            effs_.push_back(s);
        }
        for (const RigidBodyRef<3>& b : scene.rigid_bodies) {
            members_.emplace_back(b.members.begin(), b.members.end());
            std::vector<double> rest;
            for (const Vec<3>& r : b.rest_offsets)
                for (int a = 0; a < 3; a++) rest.push_back(r[a]);
            rests_.push_back(std::move(rest));
        }
        for (size_t i = 0; i < scene.rigid_bodies.size(); i++)
            rigid_.push_back({scene.rigid_bodies[i].body_id, long(members_[i].size()), members_[i].data(),
                              rests_[i].data(), scene.rigid_bodies[i].total_mass});
        for (const EmitterSpawn<3>& em : scene.emitters) {
            flume_emitter e{};
            e.particle = long(em.particle);
            e.effector = em.effector;
            for (int a = 0; a < 3; a++) {
                e.local_pos[a] = em.local_pos[a];
                e.local_vel[a] = em.local_vel[a];
            }
            emit_.push_back(e);
        }
        const size_t n = state.particles.size();
        for (const Particle<3>& p : state.particles) {
            mat_.push_back(p.material_id);
            body_.push_back(p.body_id);
            mass_.push_back(p.mass);
            vol_.push_back(p.volume0);
            act_.push_back(p.activation_substep);
        }
        desc_.n_materials = int(mats_.size());
        desc_.materials = mats_.data();
        desc_.n_effectors = int(effs_.size());
        desc_.effectors = effs_.data();
        desc_.n_rigid = int(rigid_.size());
        desc_.rigid = rigid_.data();
        desc_.n_emitters = long(emit_.size());
        desc_.emitters = emit_.data();
        desc_.n_particles = long(n);
        desc_.material_id = mat_.data();
        desc_.body_id = body_.data();
        desc_.mass = mass_.data();
        desc_.volume0 = vol_.data();
        desc_.activation_substep = act_.data();
    }

public:
    // SimState<3> (AoS, double) <-> the ABI's particle arrays (reference order); a replica
    // context gets the state repeated for every replica (the population's common start)
    void upload(const SimState<3>& st) {
        const size_t n1 = st.particles.size(), n = n1 * size_t(n_rep_);
        x_.resize(3 * n);
        v_.resize(3 * n);
        F_.resize(9 * n);
        C_.resize(9 * n);
        for (size_t i = 0; i < n; i++) {
            const Particle<3>& p = st.particles[i % n1];
            for (int a = 0; a < 3; a++) {
                x_[3 * i + a] = p.x[a];
                v_[3 * i + a] = p.v[a];
            }
            for (int r = 0; r < 3; r++)
                for (int q = 0; q < 3; q++) {
                    F_[9 * i + 3 * r + q] = p.F[r][q];
                    C_[9 * i + 3 * r + q] = p.C[r][q];
                }
        }
        const size_t ne1 = st.effectors.size();
        effst_.resize(ne1 * size_t(n_rep_));
        for (size_t k = 0; k < effst_.size(); k++) {
            const Effector<3>& e = st.effectors[k % ne1];
            for (int a = 0; a < 3; a++) {
                effst_[k].pose_t[a] = e.pose.t[a];
                effst_[k].linear_velocity[a] = e.linear_velocity[a];
                effst_[k].angular_velocity[a] = e.angular_velocity[a];
            }
            for (int r = 0; r < 3; r++)
                for (int q = 0; q < 3; q++) effst_[k].pose_R[3 * r + q] = e.pose.R[r][q];
        }
        flume_state_view view{st.time, st.substep_index, x_.data(), v_.data(), F_.data(), C_.data(), effst_.data()};
        check(ctx_, flume_state_upload(ctx_, &view));
    }

    void download(SimState<3>& st) {
        flume_state_view view{0, 0, x_.data(), v_.data(), F_.data(), C_.data(), effst_.data()};
        check(ctx_, flume_state_download(ctx_, &view));
        st.time = view.time;
        st.substep_index = view.substep_index;
        for (size_t i = 0; i < st.particles.size(); i++) {
            Particle<3>& p = st.particles[i];
            for (int a = 0; a < 3; a++) {
                p.x[a] = x_[3 * i + a];
                p.v[a] = v_[3 * i + a];
            }
            for (int r = 0; r < 3; r++)
                for (int q = 0; q < 3; q++) {
                    p.F[r][q] = F_[9 * i + 3 * r + q];
                    p.C[r][q] = C_[9 * i + 3 * r + q];
                }
        }
        for (size_t k = 0; k < st.effectors.size(); k++) {
            Effector<3>& e = st.effectors[k];
            for (int a = 0; a < 3; a++) {
                e.pose.t[a] = effst_[k].pose_t[a];
                e.linear_velocity[a] = effst_[k].linear_velocity[a];
                e.angular_velocity[a] = effst_[k].angular_velocity[a];
            }
            for (int r = 0; r < 3; r++)
                for (int q = 0; q < 3; q++) e.pose.R[r][q] = effst_[k].pose_R[3 * r + q];
        }
    }

private:
    const Scene<3>* scene_;
    int n_rep_ = 1;
    flume_ctx* ctx_ = nullptr;
    flume_scene_desc desc_{};
    std::vector<flume_material> mats_;
    std::vector<flume_effector_shape> effs_;
    std::vector<std::vector<long>> members_;
    std::vector<std::vector<double>> rests_;
    std::vector<flume_rigid_body> rigid_;
    std::vector<flume_emitter> emit_;
    std::vector<int> mat_, body_;
    std::vector<double> mass_, vol_;
    std::vector<long> act_;
    std::vector<double> x_, v_, F_, C_;
    std::vector<flume_effector_state> effst_;
};

// loss JSON (target_point / hold_initial / composite, bodies as indices, as
// build_scene rewrites them, scene.hpp:378-394) -> device loss terms
class Loss {
public:
    explicit Loss(const json& spec) {
        auto add = [&](const json& t) {
            flume_loss_term term{};
            std::string kind = t.value("kind", "target_point");
            if (kind == "target_point") {
                term.kind = FLUME_LOSS_TARGET_POINT;
                for (int a = 0; a < 3; a++) term.goal[a] = t.at("goal")[size_t(a)].get<double>();
            } else if (kind == "hold_initial") {
                term.kind = FLUME_LOSS_HOLD_INITIAL;
            } else if (kind == "mixing_spread") {
                term.kind = FLUME_LOSS_MIXING_SPREAD;
            } else if (kind == "trajectory_chamfer") {
                term.kind = FLUME_LOSS_TRAJECTORY_CHAMFER;
                std::vector<long> off{0};
                std::vector<double> pts;
                for (const json& step : t.at("goal_trajectory")) {
                    for (const json& p : step)
                        for (int a = 0; a < 3; a++) pts.push_back(p[size_t(a)].get<double>());
                    off.push_back(long(pts.size() / 3));
                }
                goal_off_.push_back(std::move(off));
                goal_pts_.push_back(std::move(pts));
                term.n_goal_steps = int(goal_off_.back().size()) - 1;
            } else {
                throw SceneError("loss kind '" + kind + "' is not evaluated on the device");
            }
            term.body = t.at("body").get<int>();
            term.weight = t.value("weight", 1.0);
            term.squared = t.value("squared", false) ? 1 : 0;
            term.final_only = t.value("eval", "per_step") == std::string("final") ? 1 : 0;
            terms_.push_back(term);
        };
        if (spec.value("kind", "") == std::string("composite"))
            for (const json& t : spec.at("terms")) add(t);
        else
            add(spec);
        // goal sets in this object's vectors (stable once all terms are parsed)
        size_t q = 0;
        for (flume_loss_term& term : terms_)
            if (term.kind == FLUME_LOSS_TRAJECTORY_CHAMFER) {
                term.goal_step_offsets = goal_off_[q].data();
                term.goal_points = goal_pts_[q].data();
                q++;
            }
        desc_ = flume_loss_desc{};
        desc_.n_terms = int(terms_.size());
        desc_.terms = terms_.data();
        desc_.attraction_body = -1;
    }
    Loss(const Loss&) = delete;
    Loss& operator=(const Loss&) = delete;
    const flume_loss_desc* desc() const { return &desc_; }

    // LossEvaluator::enable_attraction (losses.hpp:350-355)
    void enable_attraction(int body, Real weight, Real radius, Real tau) {
        desc_.attraction_body = body < 0 ? terms_.at(0).body : body;
        desc_.attraction_weight = weight;
        desc_.attraction_radius = radius;
        desc_.attraction_tau = tau;
    }
    // LossEvaluator::per_particle (losses.hpp:367-390), evaluated on the device
    std::vector<Real> per_particle(const SimState<3>& state, Workspace& ws) const {
        ws.upload(state);
        std::vector<Real> out(state.particles.size());
        check(ws.ctx(), flume_loss_per_particle(ws.ctx(), &desc_, out.data()));
        return out;
    }
    // LossEvaluator::refresh_attraction (losses.hpp:357-363)
    void refresh_attraction(const SimState<3>& state, Workspace& ws) {
        if (!(desc_.attraction_weight > 0)) return;
        std::vector<Real> all = per_particle(state, ws);
        prev_.clear();
        for (size_t i = 0; i < state.particles.size(); i++)
            if (state.particles[i].body_id == desc_.attraction_body) prev_.push_back(all[i]);
        desc_.n_prev = long(prev_.size());
        desc_.prev_losses = prev_.data();
    }

private:
    std::vector<Real> prev_;
    std::vector<flume_loss_term> terms_;
    std::vector<std::vector<long>> goal_off_;
    std::vector<std::vector<double>> goal_pts_;
    flume_loss_desc desc_{};
};

inline flume_actions actions_view(const ActionTrajectory& a, std::vector<double>& buf) {
    buf = a.flatten();
    return flume_actions{a.n_segments, a.segment_length, buf.data()};
}

// mpm.hpp:455-473
inline void mpm_substep(const Scene<3>& scene, SimState<3>& state, const std::array<Real, 6>& action,
                        Workspace& ws, int count = 1) {
    (void)scene;
    ws.upload(state);
    check(ws.ctx(), flume_substep(ws.ctx(), action.data(), count));
    ws.download(state);
}

// grad.hpp:15-41
inline Real rollout_loss(const Scene<3>& scene, const SimState<3>& state0, const ActionTrajectory& actions,
                         const Loss& loss, Workspace& ws, long window_substeps = 0,
                         std::vector<Real>* per_segment = nullptr, SimState<3>* final_state = nullptr) {
    (void)scene;
    ws.upload(state0);
    std::vector<double> buf, per(size_t(actions.n_segments));
    flume_actions av = actions_view(actions, buf);
    double out = 0;
    if (final_state) {  // the context ends on the state after the horizon
        check(ws.ctx(), flume_rollout_loss_final(ws.ctx(), &av, loss.desc(), window_substeps, &out, per.data()));
        *final_state = state0;
        ws.download(*final_state);
    } else {
        check(ws.ctx(), flume_rollout_loss(ws.ctx(), &av, loss.desc(), window_substeps, &out, per.data()));
    }
    if (per_segment) *per_segment = per;
    return out;
}

// rollout_loss of every candidate of a population in a replica context (Workspace(...,
// Replicas{n})): one kernel launch per stage for all of them; each replica's loss is the
// single-context one up to the order of its fp64 sums
inline std::vector<Real> rollout_loss_replicas(const Scene<3>& scene, const SimState<3>& state0,
                                               const std::vector<ActionTrajectory>& population, const Loss& loss,
                                               Workspace& ws, long window_substeps = 0) {
    (void)scene;
    const int R = ws.replicas();
    if (int(population.size()) != R) throw EngineError("rollout_loss_replicas: one trajectory per replica");
    const int nseg = population.front().n_segments, seglen = population.front().segment_length;
    std::vector<double> vals(size_t(nseg) * R * 6);
    for (int r = 0; r < R; r++) {
        const ActionTrajectory& a = population[size_t(r)];
        if (a.n_segments != nseg || a.segment_length != seglen)
            throw EngineError("rollout_loss_replicas: every candidate needs the same segment layout");
        for (int s = 0; s < nseg; s++)
            for (int k = 0; k < 6; k++) vals[(size_t(s) * R + r) * 6 + k] = a.values[size_t(s)][size_t(k)];
    }
    ws.upload(state0);
    flume_actions av{nseg, seglen, vals.data()};
    std::vector<Real> out(static_cast<size_t>(R), 0.0);
    check(ws.ctx(), flume_replicas_rollout_loss(ws.ctx(), &av, loss.desc(), window_substeps, 0, out.data(), nullptr));
    return out;
}

// grad.hpp:61-134
inline TrajectoryGrad<3> grad_trajectory(const Scene<3>& scene, const SimState<3>& state0,
                                         const ActionTrajectory& actions, const Loss& loss, Workspace& ws,
                                         long stride = 0, long window_substeps = 0) {
    (void)scene;
    ws.upload(state0);
    std::vector<double> buf, grad(size_t(actions.n_segments) * 6), per(size_t(actions.n_segments));
    flume_actions av = actions_view(actions, buf);
    TrajectoryGrad<3> out;
    long snaps = 0;
    check(ws.ctx(), flume_grad_trajectory(ws.ctx(), &av, loss.desc(), stride, window_substeps, grad.data(), &out.loss,
                                          &out.full_loss, per.data(), &snaps));
    out.per_segment = per;
    out.snapshots = size_t(snaps);
    out.action_grad.assign(size_t(actions.n_segments), Action6{});
    for (int s = 0; s < actions.n_segments; s++)
        for (int k = 0; k < 6; k++) out.action_grad[size_t(s)][size_t(k)] = grad[size_t(6 * s + k)];
    return out;
}

// grad.hpp:190-225: the device adjoint gradient over the optimizable components, audited
// by central differences of device rollouts (fp32 state: pick eps ~1e-3 for O(1) actions)
inline GradReport grad_check(const Scene<3>& scene, const SimState<3>& state0, const ActionTrajectory& actions,
                             const Loss& loss, Workspace& ws, long stride, Real eps, bool with_fd = true) {
    auto start = std::chrono::steady_clock::now();
    std::vector<int> comps = optimizable_components(state0);
    GradReport rep;
    TrajectoryGrad<3> tg = grad_trajectory(scene, state0, actions, loss, ws, stride);
    rep.loss = tg.loss;
    for (int s = 0; s < actions.n_segments; s++)
        for (int k : comps) rep.gradient.push_back(tg.action_grad[size_t(s)][size_t(k)]);
    if (with_fd) {
        std::vector<Real> params;
        for (int s = 0; s < actions.n_segments; s++)
            for (int k : comps) params.push_back(actions.values[size_t(s)][size_t(k)]);
        auto objective = [&](const std::vector<Real>& p) {
            ActionTrajectory a = actions;
            size_t idx = 0;
            for (int s = 0; s < a.n_segments; s++)
                for (int k : comps) a.values[size_t(s)][size_t(k)] = p[idx++];
            return rollout_loss(scene, state0, a, loss, ws);
        };
        rep.fd_gradient = finite_difference_gradient(objective, params, eps);
        rep.max_rel_error = GradReport::rel_error(rep.gradient, rep.fd_gradient);
    }
    rep.wall_time = std::chrono::duration<Real>(std::chrono::steady_clock::now() - start).count();
    return rep;
}

// adjoint.hpp:476-548 (bars of the post-state in, bars of rec.pre_state out)
inline void adjoint_substep(const Scene<3>& scene, const SubstepRecord<3>& rec, AdjointState<3>& adj,
                            std::array<Real, 6>& action_bar, Workspace& ws) {
    (void)scene;
    ws.upload(*rec.pre_state);
    const size_t n = adj.x_bar.size();
    std::vector<double> xb(3 * n), vb(3 * n), Fb(9 * n), Cb(9 * n), eb(12 * std::max<size_t>(adj.eff_t_bar.size(), 1));
    for (size_t i = 0; i < n; i++) {
        for (int a = 0; a < 3; a++) {
            xb[3 * i + a] = adj.x_bar[i][a];
            vb[3 * i + a] = adj.v_bar[i][a];
        }
        for (int r = 0; r < 3; r++)
            for (int q = 0; q < 3; q++) {
                Fb[9 * i + 3 * r + q] = adj.F_bar[i][r][q];
                Cb[9 * i + 3 * r + q] = adj.C_bar[i][r][q];
            }
    }
    for (size_t e = 0; e < adj.eff_t_bar.size(); e++) {
        for (int a = 0; a < 3; a++) eb[12 * e + a] = adj.eff_t_bar[e][a];
        for (int r = 0; r < 3; r++)
            for (int q = 0; q < 3; q++) eb[12 * e + 3 + 3 * r + q] = adj.eff_R_bar[e][r][q];
    }
    check(ws.ctx(), flume_adjoint_substep(ws.ctx(), rec.action.data(), xb.data(), vb.data(), Fb.data(), Cb.data(),
                                          eb.data(), action_bar.data()));
    for (size_t i = 0; i < n; i++) {
        for (int a = 0; a < 3; a++) {
            adj.x_bar[i][a] = xb[3 * i + a];
            adj.v_bar[i][a] = vb[3 * i + a];
        }
        for (int r = 0; r < 3; r++)
            for (int q = 0; q < 3; q++) {
                adj.F_bar[i][r][q] = Fb[9 * i + 3 * r + q];
                adj.C_bar[i][r][q] = Cb[9 * i + 3 * r + q];
            }
    }
    for (size_t e = 0; e < adj.eff_t_bar.size(); e++) {
        for (int a = 0; a < 3; a++) adj.eff_t_bar[e][a] = eb[12 * e + a];
        for (int r = 0; r < 3; r++)
            for (int q = 0; q < 3; q++) adj.eff_R_bar[e][r][q] = eb[12 * e + 3 + 3 * r + q];
    }
}

}  // namespace gpu
}  // namespace flume
