// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" driver around the *unmodified* reference engine headers
// (/root/reference/proj/include/flume/*.hpp).  Built by oracle/Makefile into
// oracle/_ref/libflume_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg / --impl reference arm may load it, as the checker
// or as the timed CPU reference -- never as the thing measured for the GPU path.
//
// Every entry point below calls the reference's own public API:
//   build_scene<3>          proj/include/flume/scene.hpp:161
//   mpm_substep<3>          proj/include/flume/mpm.hpp:455
//   p2g / grid_update       proj/include/flume/mpm.hpp:249 / :301
//   adjoint_substep<3>      proj/include/flume/adjoint.hpp:476
//   rollout_loss            proj/include/flume/grad.hpp:15
//   grad_trajectory         proj/include/flume/grad.hpp:61
//   LossEvaluator           proj/include/flume/losses.hpp:306
// 3D only (the GPU path is 3D).
#include <cstring>
#include <memory>
#include <string>

#include "flume/flume.hpp"
#include "flume/io.hpp"

using namespace flume;

namespace {

struct RefWorld {
    World<3> w;
    SimState<3> state;  // the live state the calls mutate
    MpmWorkspace<3> ws;
    // attraction (LossEvaluator::enable_attraction / refresh_attraction, losses.hpp:350-363)
    bool att_on = false;
    int att_body = -1;
    Real att_weight = 0, att_radius = 0, att_tau = 0;
    SimState<3> att_refresh;  // the state refresh_attraction reads
};

// the LossEvaluator a call uses: built from the live state like the reference's
// drivers do, with the attraction term enabled and refreshed when configured
std::unique_ptr<LossEvaluator<3>> make_le(RefWorld* rw) {
    auto le = std::make_unique<LossEvaluator<3>>(rw->w.scene, rw->w.loss_spec, rw->state);
    if (rw->att_on) {
        le->enable_attraction(rw->att_body, rw->att_weight, rw->att_radius, rw->att_tau);
        le->refresh_attraction(rw->att_refresh);
    }
    return le;
}

thread_local std::string g_err;
thread_local long g_err_pid = -1;
thread_local long g_err_body = -1;
thread_local long g_err_substep = -1;

// error codes shared with paper_2303_02346_b200 (include/flume_b200.h)
enum { OK = 0, E_ENGINE = 1, E_SCENE = 2, E_DEGENERATE = 3, E_RIGIDITY = 4, E_ADJOINT = 5,
       E_SOLVER = 6, E_OTHER = 9 };

template <typename F>
int guarded(F&& f) {
    g_err.clear();
    g_err_pid = g_err_body = g_err_substep = -1;
    try {
        f();
        return OK;
    } catch (const SceneError& e) {
        g_err = e.what();
        return E_SCENE;
    } catch (const DegenerateDeformation& e) {
        g_err = e.what();
        g_err_pid = e.particle_id;
        return E_DEGENERATE;
    } catch (const RigidityError& e) {
        g_err = e.what();
        g_err_body = e.body_id;
        return E_RIGIDITY;
    } catch (const AdjointError& e) {
        g_err = e.what();
        g_err_substep = e.substep;
        return E_ADJOINT;
    } catch (const SolverError& e) {
        g_err = e.what();
        return E_SOLVER;
    } catch (const EngineError& e) {
        g_err = e.what();
        return E_ENGINE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return E_OTHER;
    }
}

ActionTrajectory make_actions(int nseg, int seglen, const double* values) {
    ActionTrajectory a(nseg, seglen);
    for (int s = 0; s < nseg; s++)
        for (int k = 0; k < 6; k++) a.values[size_t(s)][size_t(k)] = values[s * 6 + k];
    return a;
}

}  // namespace

extern "C" {

const char* ref_last_error(long* pid, long* body, long* substep) {
    if (pid) *pid = g_err_pid;
    if (body) *body = g_err_body;
    if (substep) *substep = g_err_substep;
    return g_err.c_str();
}

int ref_world_from_json(const char* text, void** out) {
    *out = nullptr;
    return guarded([&] {
        json spec = json::parse(text);
        auto rw = std::make_unique<RefWorld>();
        rw->w = build_scene<3>(spec);
        rw->state = rw->w.state;
        *out = rw.release();
    });
}

void ref_world_free(void* h) { delete static_cast<RefWorld*>(h); }

long ref_num_particles(void* h) { return long(static_cast<RefWorld*>(h)->state.particles.size()); }
int ref_num_effectors(void* h) { return int(static_cast<RefWorld*>(h)->state.effectors.size()); }
int ref_num_materials(void* h) { return int(static_cast<RefWorld*>(h)->w.scene.materials.size()); }
int ref_num_rigid(void* h) { return int(static_cast<RefWorld*>(h)->w.scene.rigid_bodies.size()); }
long ref_num_emitters(void* h) { return long(static_cast<RefWorld*>(h)->w.scene.emitters.size()); }

// config: res, dims[3] | dt, dx, domain[3], gravity[3], contact_eps, cfl, mass_eps | bw, hard
void ref_config(void* h, int* ints, double* reals) {
    const SimConfig<3>& c = static_cast<RefWorld*>(h)->w.scene.config;
    IVec<3> d = c.node_dims();
    ints[0] = c.grid_resolution;
    ints[1] = d[0];
    ints[2] = d[1];
    ints[3] = d[2];
    ints[4] = c.boundary_width;
    ints[5] = c.hard_contact ? 1 : 0;
    ints[6] = c.substeps_per_step;
    reals[0] = c.dt_substep;
    reals[1] = c.dx();
    for (int a = 0; a < 3; a++) reals[2 + a] = c.domain_extent[a];
    for (int a = 0; a < 3; a++) reals[5 + a] = c.gravity[a];
    reals[8] = c.contact_eps_cells;
    reals[9] = c.cfl_fraction;
    reals[10] = c.mass_epsilon;
}

void ref_set_hard_contact(void* h, int hard) {
    static_cast<RefWorld*>(h)->w.scene.config.hard_contact = hard != 0;
}

void ref_set_gravity(void* h, const double* g) {
    for (int a = 0; a < 3; a++) static_cast<RefWorld*>(h)->w.scene.config.gravity[a] = g[a];
}

// kind, mu, lambda, rho, theta_c, theta_s, sigma_y  (7 doubles per material)
void ref_materials(void* h, double* out) {
    const auto& ms = static_cast<RefWorld*>(h)->w.scene.materials;
    for (size_t i = 0; i < ms.size(); i++) {
        double* o = out + 7 * i;
        o[0] = double(int(ms[i].kind));
        o[1] = ms[i].mu;
        o[2] = ms[i].lambda;
        o[3] = ms[i].rho;
        o[4] = ms[i].yield.theta_c;
        o[5] = ms[i].yield.theta_s;
        o[6] = ms[i].yield.sigma_y;
    }
}

// Effector record (64 doubles): kind, radius, half[3], seg_a[3], seg_b[3], normal[3], offset,
// half_height, shape_t[3], shape_R[9], pose_t[3], pose_R[9], lin[3], ang[3], mu, mask[6]
void ref_effectors(void* h, double* out) {
    const auto& es = static_cast<RefWorld*>(h)->state.effectors;
    for (size_t i = 0; i < es.size(); i++) {
        const Effector<3>& e = es[i];
        double* o = out + 64 * i;
        int k = 0;
        o[k++] = double(int(e.sdf.shape.kind));
        o[k++] = e.sdf.shape.radius;
        for (int a = 0; a < 3; a++) o[k++] = e.sdf.shape.half_extents[a];
        for (int a = 0; a < 3; a++) o[k++] = e.sdf.shape.seg_a[a];
        for (int a = 0; a < 3; a++) o[k++] = e.sdf.shape.seg_b[a];
        for (int a = 0; a < 3; a++) o[k++] = e.sdf.shape.plane_normal[a];
        o[k++] = e.sdf.shape.plane_offset;
        o[k++] = e.sdf.shape.half_height;
        for (int a = 0; a < 3; a++) o[k++] = e.sdf.pose.t[a];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) o[k++] = e.sdf.pose.R[r][c];
        for (int a = 0; a < 3; a++) o[k++] = e.pose.t[a];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) o[k++] = e.pose.R[r][c];
        for (int a = 0; a < 3; a++) o[k++] = e.linear_velocity[a];
        for (int a = 0; a < 3; a++) o[k++] = e.angular_velocity[a];
        o[k++] = e.friction_mu;
        for (int a = 0; a < 6; a++) o[k++] = e.action_mask[size_t(a)] ? 1.0 : 0.0;
    }
}

long ref_rigid_members(void* h, int body, long* members, double* rest, int* body_id,
                       double* total_mass) {
    const auto& rb = static_cast<RefWorld*>(h)->w.scene.rigid_bodies[size_t(body)];
    if (members)
        for (size_t j = 0; j < rb.members.size(); j++) {
            members[j] = long(rb.members[j]);
            for (int a = 0; a < 3; a++) rest[3 * j + a] = rb.rest_offsets[j][a];
        }
    if (body_id) *body_id = rb.body_id;
    if (total_mass) *total_mass = rb.total_mass;
    return long(rb.members.size());
}

// particle, effector, local_pos[3], local_vel[3]
void ref_emitters(void* h, long* particle, int* effector, double* local_pos, double* local_vel) {
    const auto& em = static_cast<RefWorld*>(h)->w.scene.emitters;
    for (size_t i = 0; i < em.size(); i++) {
        particle[i] = long(em[i].particle);
        effector[i] = em[i].effector;
        for (int a = 0; a < 3; a++) {
            local_pos[3 * i + a] = em[i].local_pos[a];
            local_vel[3 * i + a] = em[i].local_vel[a];
        }
    }
}

const char* ref_loss_spec(void* h) {
    static thread_local std::string s;
    s = static_cast<RefWorld*>(h)->w.loss_spec.dump();
    return s.c_str();
}
// versioned state snapshots (io.hpp:144-240)
const char* ref_snapshot_dump(void* h) {
    static thread_local std::string s;
    s = state_to_json<3>(static_cast<RefWorld*>(h)->state).dump();
    return s.c_str();
}
int ref_snapshot_load(void* h, const char* text) {
    try {
        state_from_json<3>(json::parse(text), static_cast<RefWorld*>(h)->state);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
const char* ref_optimizer_spec(void* h) {
    static thread_local std::string s;
    s = static_cast<RefWorld*>(h)->w.optimizer_spec.dump();
    return s.c_str();
}

// Particle arrays; any pointer may be null.  F and C row-major 9 per particle.
void ref_get_state(void* h, double* x, double* v, double* F, double* C, double* mass,
                   double* vol0, int* mat, int* body, long* act, double* time, long* substep) {
    const SimState<3>& st = static_cast<RefWorld*>(h)->state;
    for (size_t i = 0; i < st.particles.size(); i++) {
        const Particle<3>& p = st.particles[i];
        for (int a = 0; a < 3; a++) {
            if (x) x[3 * i + a] = p.x[a];
            if (v) v[3 * i + a] = p.v[a];
        }
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) {
                if (F) F[9 * i + 3 * r + c] = p.F[r][c];
                if (C) C[9 * i + 3 * r + c] = p.C[r][c];
            }
        if (mass) mass[i] = p.mass;
        if (vol0) vol0[i] = p.volume0;
        if (mat) mat[i] = p.material_id;
        if (body) body[i] = p.body_id;
        if (act) act[i] = p.activation_substep;
    }
    if (time) *time = st.time;
    if (substep) *substep = st.substep_index;
}

void ref_set_state(void* h, const double* x, const double* v, const double* F, const double* C,
                   const double* mass, const double* vol0, const int* mat, const int* body,
                   const long* act, const double* time, const long* substep) {
    SimState<3>& st = static_cast<RefWorld*>(h)->state;
    for (size_t i = 0; i < st.particles.size(); i++) {
        Particle<3>& p = st.particles[i];
        for (int a = 0; a < 3; a++) {
            if (x) p.x[a] = x[3 * i + a];
            if (v) p.v[a] = v[3 * i + a];
        }
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) {
                if (F) p.F[r][c] = F[9 * i + 3 * r + c];
                if (C) p.C[r][c] = C[9 * i + 3 * r + c];
            }
        if (mass) p.mass = mass[i];
        if (vol0) p.volume0 = vol0[i];
        if (mat) p.material_id = mat[i];
        if (body) p.body_id = body[i];
        if (act) p.activation_substep = act[i];
    }
    if (time) st.time = *time;
    if (substep) st.substep_index = *substep;
}

// effector dynamic state: pose_t[3], pose_R[9], lin[3], ang[3] per effector (18 doubles)
void ref_get_effector_state(void* h, double* out) {
    const auto& es = static_cast<RefWorld*>(h)->state.effectors;
    for (size_t i = 0; i < es.size(); i++) {
        double* o = out + 18 * i;
        for (int a = 0; a < 3; a++) o[a] = es[i].pose.t[a];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) o[3 + 3 * r + c] = es[i].pose.R[r][c];
        for (int a = 0; a < 3; a++) o[12 + a] = es[i].linear_velocity[a];
        for (int a = 0; a < 3; a++) o[15 + a] = es[i].angular_velocity[a];
    }
}

void ref_set_effector_state(void* h, const double* in) {
    auto& es = static_cast<RefWorld*>(h)->state.effectors;
    for (size_t i = 0; i < es.size(); i++) {
        const double* o = in + 18 * i;
        for (int a = 0; a < 3; a++) es[i].pose.t[a] = o[a];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) es[i].pose.R[r][c] = o[3 + 3 * r + c];
        for (int a = 0; a < 3; a++) es[i].linear_velocity[a] = o[12 + a];
        for (int a = 0; a < 3; a++) es[i].angular_velocity[a] = o[15 + a];
    }
}

void ref_reset_state(void* h) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    rw->state = rw->w.state;
}

int ref_substep(void* h, const double* action, int count) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        std::array<Real, 6> a{};
        for (int k = 0; k < 6; k++) a[size_t(k)] = action[k];
        for (int i = 0; i < count; i++) mpm_substep(rw->w.scene, rw->state, a, rw->ws);
    });
}

// p2g + grid_update on the live state (no advance); dense node grids, flat
// index (i*ny + j)*nz + k as in grid.hpp:32-36.
int ref_p2g_grid(void* h, double* mass, double* mom, double* vel) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        p2g(rw->w.scene, rw->state, rw->ws);
        if (mom)
            for (size_t i = 0; i < rw->ws.mom.size(); i++)
                for (int a = 0; a < 3; a++) mom[3 * i + a] = rw->ws.mom.data[i][a];
        grid_update(rw->w.scene, rw->state, rw->ws);
        for (size_t i = 0; i < rw->ws.mass.size(); i++) {
            if (mass) mass[i] = rw->ws.mass.data[i];
            if (vel)
                for (int a = 0; a < 3; a++) vel[3 * i + a] = rw->ws.vel.data[i][a];
        }
    });
}

int ref_rollout_loss(void* h, int nseg, int seglen, const double* actions, long window,
                     double* loss, double* per_segment) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        ActionTrajectory a = make_actions(nseg, seglen, actions);
        auto le = make_le(rw);
        std::vector<Real> per;
        *loss = rollout_loss(rw->w.scene, rw->state, a, *le, window, &per);
        if (per_segment)
            for (int s = 0; s < nseg; s++) per_segment[s] = per[size_t(s)];
    });
}

int ref_grad_trajectory(void* h, int nseg, int seglen, const double* actions, long stride,
                        long window, double* grad, double* loss, double* full_loss,
                        double* per_segment, long* snapshots) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        ActionTrajectory a = make_actions(nseg, seglen, actions);
        auto le = make_le(rw);
        TrajectoryGrad<3> tg = grad_trajectory(rw->w.scene, rw->state, a, *le, stride, window);
        for (int s = 0; s < nseg; s++)
            for (int k = 0; k < 6; k++) grad[s * 6 + k] = tg.action_grad[size_t(s)][size_t(k)];
        if (loss) *loss = tg.loss;
        if (full_loss) *full_loss = tg.full_loss;
        if (per_segment)
            for (int s = 0; s < nseg; s++) per_segment[s] = tg.per_segment[size_t(s)];
        if (snapshots) *snapshots = long(tg.snapshots);
    });
}

// grad_check (grad.hpp:190-225): adjoint gradient over the optimizable components and,
// with_fd, its central-difference audit; arrays hold up to nseg * 6 entries
int ref_grad_check(void* h, int nseg, int seglen, const double* actions, long stride, double eps, int with_fd,
                   double* grad, double* fd, long* n, double* max_rel, double* loss) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        ActionTrajectory a = make_actions(nseg, seglen, actions);
        auto le = make_le(rw);
        GradReport rep = grad_check(rw->w.scene, rw->state, a, *le, stride, eps, with_fd != 0);
        *n = long(rep.gradient.size());
        for (size_t i = 0; i < rep.gradient.size(); i++) grad[i] = rep.gradient[i];
        for (size_t i = 0; i < rep.fd_gradient.size(); i++) fd[i] = rep.fd_gradient[i];
        *max_rel = rep.max_rel_error;
        *loss = rep.loss;
    });
}

// run outputs (io.hpp:53-114) of the live state
int ref_write_frame_csv(void* h, const char* path, unsigned long long hash) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] { write_frame_csv<3>(path, rw->state, hash); });
}
int ref_write_metrics(void* h, const char* path, unsigned long long hash) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        MetricsWriter<3> m(path, hash);
        m.append(rw->state);
        m.flush();
    });
}
const char* ref_actions_json(int nseg, int seglen, const double* values) {
    static thread_local std::string s;
    s = actions_to_json(make_actions(nseg, seglen, values)).dump();
    return s.c_str();
}

// Attraction for the following rollout_loss / grad_trajectory calls: weight <= 0 turns it
// off; refresh_x (n*3) = positions of the state refresh_attraction reads (the live state
// with x replaced)
void ref_set_attraction(void* h, int body, double weight, double radius, double tau, const double* refresh_x) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    rw->att_on = weight > 0;
    rw->att_body = body;
    rw->att_weight = weight;
    rw->att_radius = radius;
    rw->att_tau = tau;
    rw->att_refresh = rw->state;
    if (refresh_x)
        for (size_t i = 0; i < rw->att_refresh.particles.size(); i++)
            for (int a = 0; a < 3; a++) rw->att_refresh.particles[i].x[a] = refresh_x[3 * i + a];
}

// LossEvaluator::per_particle (losses.hpp:367) of the live state with x replaced by xs (n*3) if given
int ref_per_particle(void* h, const double* xs, double* out) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        LossEvaluator<3> le(rw->w.scene, rw->w.loss_spec, rw->state);
        SimState<3> st = rw->state;
        if (xs)
            for (size_t i = 0; i < st.particles.size(); i++)
                for (int a = 0; a < 3; a++) st.particles[i].x[a] = xs[3 * i + a];
        std::vector<Real> v = le.per_particle(st);
        for (size_t i = 0; i < v.size(); i++) out[i] = v[i];
    });
}

// One adjoint substep from the live state (the pre-state), reference adjoint.hpp:476.
// Bars are per particle (x,v: 3; F,C: 9 row-major) and are read and overwritten.
// eff_bars: per effector t_bar[3], R_bar[9] (read/overwritten).  action_bar[6] accumulates.
int ref_adjoint_substep(void* h, const double* action, double* xb, double* vb, double* Fb,
                        double* Cb, double* eff_bars, double* action_bar) {
    RefWorld* rw = static_cast<RefWorld*>(h);
    return guarded([&] {
        AdjointState<3> adj;
        adj.init(rw->state);
        size_t n = rw->state.particles.size();
        for (size_t i = 0; i < n; i++) {
            for (int a = 0; a < 3; a++) {
                adj.x_bar[i][a] = xb[3 * i + a];
                adj.v_bar[i][a] = vb[3 * i + a];
            }
            for (int r = 0; r < 3; r++)
                for (int c = 0; c < 3; c++) {
                    adj.F_bar[i][r][c] = Fb[9 * i + 3 * r + c];
                    adj.C_bar[i][r][c] = Cb[9 * i + 3 * r + c];
                }
        }
        for (size_t e = 0; e < adj.eff_t_bar.size(); e++) {
            for (int a = 0; a < 3; a++) adj.eff_t_bar[e][a] = eff_bars[12 * e + a];
            for (int r = 0; r < 3; r++)
                for (int c = 0; c < 3; c++) adj.eff_R_bar[e][r][c] = eff_bars[12 * e + 3 + 3 * r + c];
        }
        std::array<Real, 6> act{}, abar{};
        for (int k = 0; k < 6; k++) {
            act[size_t(k)] = action[k];
            abar[size_t(k)] = action_bar[k];
        }
        SubstepRecord<3> rec{rw->state.substep_index, act, &rw->state};
        adjoint_substep(rw->w.scene, rec, adj, abar, rw->ws);
        for (size_t i = 0; i < n; i++) {
            for (int a = 0; a < 3; a++) {
                xb[3 * i + a] = adj.x_bar[i][a];
                vb[3 * i + a] = adj.v_bar[i][a];
            }
            for (int r = 0; r < 3; r++)
                for (int c = 0; c < 3; c++) {
                    Fb[9 * i + 3 * r + c] = adj.F_bar[i][r][c];
                    Cb[9 * i + 3 * r + c] = adj.C_bar[i][r][c];
                }
        }
        for (size_t e = 0; e < adj.eff_t_bar.size(); e++) {
            for (int a = 0; a < 3; a++) eff_bars[12 * e + a] = adj.eff_t_bar[e][a];
            for (int r = 0; r < 3; r++)
                for (int c = 0; c < 3; c++) eff_bars[12 * e + 3 + 3 * r + c] = adj.eff_R_bar[e][r][c];
        }
        for (int k = 0; k < 6; k++) action_bar[k] = abar[size_t(k)];
    });
}

}  // extern "C"
