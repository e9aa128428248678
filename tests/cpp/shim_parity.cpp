// tests/cpp/shim_parity.cpp -- TEST INFRASTRUCTURE: the reference engine's own C++
// API (proj/include/flume) next to the drop-in adapter include/flume/gpu.hpp.
// Builds one scene with the reference's build_scene<3>, advances a copy of the
// state with flume::mpm_substep (CPU, fp64) and with flume::gpu::mpm_substep
// (B200), then compares grad_trajectory from both.  Prints one JSON line;
// exit code 0 when within the parity tolerances of tests/test_gpu_forward.py.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "flume/flume.hpp"
#include "flume/gpu.hpp"

using namespace flume;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: shim_parity scene.json [substeps]\n");
        return 2;
    }
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    json spec = json::parse(ss.str());
    const int steps = argc > 2 ? std::atoi(argv[2]) : 5;
    World<3> w = build_scene<3>(spec);
    std::array<Real, 6> act{};
    for (int k = 0; k < 6; k++) act[size_t(k)] = spec["optimizer"]["init"][size_t(k)].get<double>();

    SimState<3> cpu = w.state, dev = w.state;
    MpmWorkspace<3> mws;
    gpu::Workspace gws(w.scene, w.state, 0);
    for (int t = 0; t < steps; t++) mpm_substep(w.scene, cpu, act, mws);
    gpu::mpm_substep(w.scene, dev, act, gws, steps);
    double dx = 0, dv = 0, vmax = 0;
    for (size_t i = 0; i < cpu.particles.size(); i++)
        for (int a = 0; a < 3; a++) {
            dx = std::max(dx, std::abs(cpu.particles[i].x[a] - dev.particles[i].x[a]));
            dv = std::max(dv, std::abs(cpu.particles[i].v[a] - dev.particles[i].v[a]));
            vmax = std::max(vmax, std::abs(cpu.particles[i].v[a]));
        }
    dx /= w.scene.config.dx();

    ActionTrajectory traj(2, 3);
    traj.values[0] = act;
    traj.values[1] = act;
    LossEvaluator<3> le(w.scene, w.loss_spec, w.state);
    TrajectoryGrad<3> gc = grad_trajectory(w.scene, w.state, traj, le, 2);
    TrajectoryGrad<3> gg = gpu::grad_trajectory(w.scene, w.state, traj, gpu::Loss(w.loss_spec), gws, 2);
    double gnum = 0, gden = 0;
    for (int s = 0; s < 2; s++)
        for (int k = 0; k < 6; k++) {
            gnum = std::max(gnum, std::abs(gc.action_grad[size_t(s)][size_t(k)] - gg.action_grad[size_t(s)][size_t(k)]));
            gden = std::max(gden, std::abs(gc.action_grad[size_t(s)][size_t(k)]));
        }
    const double grel = gnum / (gden + 1e-12);
    // rollout_loss's final_state: the state after the horizon equals the substep chain
    SimState<3> fin_c, fin_g;
    rollout_loss(w.scene, w.state, traj, le, 0, nullptr, &fin_c);
    gpu::Loss fl_loss(w.loss_spec);
    gpu::rollout_loss(w.scene, w.state, traj, fl_loss, gws, 0, nullptr, &fin_g);
    double fdx = 0;
    for (size_t i = 0; i < fin_c.particles.size(); i++)
        for (int a = 0; a < 3; a++) fdx = std::max(fdx, std::abs(fin_c.particles[i].x[a] - fin_g.particles[i].x[a]));
    fdx /= w.scene.config.dx();
    const bool fin_ok = fin_g.substep_index == fin_c.substep_index && fdx <= 1e-4;
    // grad_check without the FD audit: the gradient over the optimizable components
    gpu::Loss gl(w.loss_spec);
    GradReport rc = grad_check(w.scene, w.state, traj, le, 2, 1e-5, false);
    GradReport rg = gpu::grad_check(w.scene, w.state, traj, gl, gws, 2, 1e-3, false);
    const double crel = rc.gradient.size() == rg.gradient.size() ? GradReport::rel_error(rg.gradient, rc.gradient) : 1.0;
    const double lrel = std::abs(gc.loss - gg.loss) / std::abs(gc.loss);
    // a two-candidate population in one replica context against single-context rollouts
    ActionTrajectory traj2 = traj;
    for (auto& v : traj2.values)
        for (auto& c : v) c *= 0.5;
    gpu::Workspace rws(w.scene, w.state, gpu::Replicas{2}, 0);
    const std::vector<Real> pl = gpu::rollout_loss_replicas(w.scene, w.state, {traj, traj2}, fl_loss, rws);
    const Real l0 = gpu::rollout_loss(w.scene, w.state, traj, fl_loss, gws);
    const Real l1 = gpu::rollout_loss(w.scene, w.state, traj2, fl_loss, gws);
    const double prel = std::max(std::abs(pl[0] - l0) / std::abs(l0), std::abs(pl[1] - l1) / std::abs(l1));
    const bool ok = dx <= 1e-4 && dv <= 5e-4 * vmax && grel <= 1e-3 && crel <= 1e-3 && fin_ok && lrel <= 1e-5 &&
                    gc.snapshots == gg.snapshots && prel <= 1e-12;
    std::printf("{\"particles\": %zu, \"substeps\": %d, \"x_err_dx\": %.3e, \"v_err_rel\": %.3e, "
                "\"loss_rel\": %.3e, \"grad_rel\": %.3e, \"grad_check_rel\": %.3e, \"snapshots\": [%zu, %zu], "
                "\"replica_loss_rel\": %.3e, \"ok\": %s}\n",
                cpu.particles.size(), steps, dx, dv / vmax, lrel, grel, crel, gc.snapshots, gg.snapshots, prel,
                ok ? "true" : "false");
    return ok ? 0 : 1;
}
