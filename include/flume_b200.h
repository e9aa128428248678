/* flume_b200.h -- C ABI of the B200-native differentiable MLS-MPM substep.
 *
 * This is the drop-in boundary for the reference engine's hot path
 * (proj/include/flume, header-only C++20).  The reference has no FFI; its
 * "API" is the set of templated C++ calls below, and each entry point here
 * replaces one of them for D = 3 (the C++ adapter include/flume/gpu.hpp
 * re-exposes the reference signatures on top of this ABI):
 *
 *   flume_ctx_create / flume_state_upload / flume_state_download
 *       Scene<3> + SimState<3> hand-off        types.hpp:179-235, scene.hpp:161
 *   flume_substep                               mpm_substep      mpm.hpp:455-473
 *   flume_stage_grid                            p2g + grid_update mpm.hpp:249-320
 *   flume_adjoint_substep                       adjoint_substep  adjoint.hpp:476-548
 *   flume_rollout_loss                          rollout_loss     grad.hpp:15-41
 *   flume_rollout_loss_final                    rollout_loss(..., final_state) grad.hpp:15-41
 *   flume_loss_per_particle                     LossEvaluator::per_particle losses.hpp:367
 *   flume_grad_trajectory                       grad_trajectory  grad.hpp:61-134
 *                                               (+ CheckpointStore checkpoint.hpp:11-50)
 *   flume_set_mode                              SimConfig::hard_contact types.hpp:65
 *   flume_last_error                            EngineError hierarchy core.hpp:18-48
 *   flume_scene_build_json (+ accessors)        build_scene<3>   scene.hpp:161-408
 *
 * Conventions: plain pointers and sizes, no C++ or torch types; particle
 * arrays are in the reference's particle index order ("id"), row-major per
 * particle (x,v: n*3; F,C: n*9).  Every call returns a flume_status; on
 * failure flume_last_error() carries the reference exception's context.
 * A context is single-threaded; distinct contexts are
 * independent.  Execution is always deterministic: reruns are bit-identical.
 */
#ifndef FLUME_B200_H
#define FLUME_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define FLUME_B200_ABI_VERSION 3

typedef enum {
    FLUME_OK = 0,
    FLUME_E_ENGINE = 1,      /* EngineError        core.hpp:18 */
    FLUME_E_SCENE = 2,       /* SceneError         core.hpp:22 */
    FLUME_E_DEGENERATE = 3,  /* DegenerateDeformation core.hpp:26 (particle_id) */
    FLUME_E_RIGIDITY = 4,    /* RigidityError      core.hpp:32 (body_id) */
    FLUME_E_ADJOINT = 5,     /* AdjointError       core.hpp:44 (substep) */
    FLUME_E_SOLVER = 6,      /* SolverError        core.hpp:38 */
    FLUME_E_CUDA = 7,        /* device / driver failure */
    FLUME_E_ARG = 8,         /* invalid argument */
    FLUME_E_OTHER = 9
} flume_status;

typedef struct flume_ctx flume_ctx;
typedef struct flume_scene flume_scene;

/* SimConfig<3> (types.hpp:53-95) */
typedef struct {
    int grid_resolution;
    double domain[3];
    double dt_substep;
    int substeps_per_step;
    double gravity[3];
    int boundary_width;
    double contact_eps_cells;
    double cfl_fraction;
    double mass_epsilon;
    int hard_contact;
} flume_config;

/* MaterialParams (types.hpp:32-51); kind numbering = MaterialKind */
typedef struct {
    int kind;
    double mu, lambda, rho;
    double theta_c, theta_s, sigma_y;
} flume_material;

/* static part of Effector<3> (types.hpp:114-125, sdf.hpp:37-73);
 * shape_kind numbering = ShapeKind; friction_mu = +inf means sticky */
typedef struct {
    int shape_kind;
    double radius;
    double half_extents[3];
    double seg_a[3], seg_b[3];
    double plane_normal[3];
    double plane_offset;
    double half_height;
    double shape_t[3];
    double shape_R[9];
    double friction_mu;
    int action_mask[6];
} flume_effector_shape;

/* dynamic part of Effector<3> */
typedef struct {
    double pose_t[3];
    double pose_R[9];
    double linear_velocity[3];
    double angular_velocity[3];
} flume_effector_state;

/* RigidBodyRef<3> (types.hpp:218-224) */
typedef struct {
    int body_id;
    long n_members;
    const long* members;
    const double* rest_offsets; /* n_members*3 */
    double total_mass;
} flume_rigid_body;

/* EmitterSpawn<3> (types.hpp:209-215) */
typedef struct {
    long particle;
    int effector;
    double local_pos[3];
    double local_vel[3];
} flume_emitter;

/* Scene<3> plus the immutable per-particle fields of SimState<3> */
typedef struct {
    flume_config config;
    int n_materials;
    const flume_material* materials;
    int n_effectors;
    const flume_effector_shape* effectors;
    int n_rigid;
    const flume_rigid_body* rigid;
    long n_emitters;
    const flume_emitter* emitters;
    long n_particles;
    const int* material_id;
    const int* body_id;
    const double* mass;
    const double* volume0;
    const long* activation_substep;
} flume_scene_desc;

/* mutable part of SimState<3> */
typedef struct {
    double time;
    long substep_index;
    double* x; /* n*3 */
    double* v; /* n*3 */
    double* F; /* n*9 */
    double* C; /* n*9 */
    flume_effector_state* effectors; /* n_effectors */
} flume_state_view;

/* LossEvaluator terms supported on device (losses.hpp:474-551) */
/* LossTerm kinds (losses.hpp:293-304, 405-441); air_sensors needs the gas solver (out of scope) */
typedef enum {
    FLUME_LOSS_TARGET_POINT = 0,
    FLUME_LOSS_HOLD_INITIAL = 1,
    FLUME_LOSS_MIXING_SPREAD = 2,      /* -sum_ij |x_i - x_j| over the body, O(N^2) on the device */
    FLUME_LOSS_TRAJECTORY_CHAMFER = 3  /* symmetric mean nearest-neighbour distance to goal sets */
} flume_loss_kind;
typedef struct {
    int kind;
    int body;
    double weight;
    int squared;
    int final_only;
    double goal[3];
    /* trajectory_chamfer: point set s = goal_points[3*goal_step_offsets[s] .. 3*goal_step_offsets[s+1]);
       segment seg uses set min(seg, n_goal_steps - 1) (losses.hpp:488-491) */
    int n_goal_steps;
    const long* goal_step_offsets; /* n_goal_steps + 1 */
    const double* goal_points;
} flume_loss_term;
typedef struct {
    int n_terms;
    const flume_loss_term* terms;
    /* attraction term: the optimizer's gradient-sharing surrogate, added at every segment
       boundary (LossEvaluator::enable_attraction / refresh_attraction, losses.hpp:348-363;
       attraction_loss, losses.hpp:168-218).  On when attraction_weight > 0 and n_prev > 0.
       Single-rank contexts only. */
    int attraction_body;       /* < 0: the first term's body (primary_body) */
    double attraction_weight;
    double attraction_radius;  /* world units (optimize_dp passes 3 dx when its config says 0) */
    double attraction_tau;     /* <= 0: max(0.1 * median(prev_losses), 1e-9) */
    long n_prev;               /* must equal the body's member count (else FLUME_E_ENGINE) */
    const double* prev_losses; /* previous iterate's per_particle losses, body members in id order */
} flume_loss_desc;

/* ActionTrajectory (actions.hpp:13-39): values = n_segments*6 */
typedef struct {
    int n_segments;
    int segment_length;
    const double* values;
} flume_actions;

typedef struct {
    int code;
    long particle_id;
    int body_id;
    long substep;
    char message[256];
} flume_error_info;

/* per-call timing breakdown (device ms, CUDA events on the context stream) */
typedef struct {
    double forward_ms;
    double backward_ms;
    long substeps;
    long particle_substeps;
    long launches;
} flume_timing;

int flume_abi_version(void);

/* ---- scene construction (build_scene<3>, scene.hpp:161-408) ---- */
int flume_scene_build_json(const char* json_text, flume_scene** out);
int flume_scene_free(flume_scene* s);
int flume_scene_desc_get(const flume_scene* s, flume_scene_desc* out); /* pointers owned by s */
int flume_scene_state_get(const flume_scene* s, flume_state_view* out); /* initial state, owned by s */
int flume_scene_loss_get(const flume_scene* s, flume_loss_desc* out);
int flume_scene_optimizer_get(const flume_scene* s, int* n_segments, int* segment_length, double* init6);

/* ---- context ---- */
int flume_ctx_create(const flume_scene_desc* desc, int device, flume_ctx** out);
/* ---- replica contexts (a CMA-ES population, optimize.hpp:383-418) ----
 * n_replicas copies of one scene side by side in one grid (one empty 4-cell column between
 * them; positions stay replica-local), so every kernel launch of a substep covers the whole
 * population.  Particle i of replica r is r * n_particles + i and effector e is
 * r * n_effectors + e in every state view (flume_state_upload / download take the
 * concatenated arrays); body b is r * body_stride + b.  flume_substep takes n_replicas x 6
 * action values.  Each replica's state evolves bit-identically to a single context's.
 * adjoint_substep, stage_grid and loss_per_particle return FLUME_E_ARG, and so do the single
 * rollout / gradient entry points (use the flume_replicas_* ones). */
int flume_ctx_create_replicas(const flume_scene_desc* desc, int n_replicas, int device, flume_ctx** out);
/* rollout_loss (grad.hpp:15-41) of every replica: actions->values = n_segments x n_replicas x 6
 * (segment-major), `loss` is the scene's own description (applied to each replica's bodies);
 * loss_out[n_replicas], per_segment[n_replicas x n_segments] (may be NULL).  keep_final != 0:
 * the context continues from the final states (flume_rollout_loss_final). */
int flume_replicas_rollout_loss(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss,
                                long window, int keep_final, double* loss_out, double* per_segment);
/* grad_trajectory (grad.hpp:61-134) of every replica (a population of independent
 * gradient-based optimizations, optimize.hpp:180-239): action_grad[n_replicas x n_segments x 6],
 * loss_out / full_loss[n_replicas], per_segment[n_replicas x n_segments]; actions and loss as
 * in flume_replicas_rollout_loss. */
int flume_replicas_grad_trajectory(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss,
                                   long stride, long window, double* action_grad, double* loss_out,
                                   double* full_loss, double* per_segment, long* snapshots);
int flume_replicas_info(const flume_ctx* ctx, int* n_replicas, long* particles_per_replica,
                        int* effectors_per_replica, int* body_stride);
int flume_ctx_destroy(flume_ctx* ctx);
int flume_set_mode(flume_ctx* ctx, int deterministic, int hard_contact);
int flume_last_error(const flume_ctx* ctx, flume_error_info* info);
/* CheckpointStore placement for grad_trajectory (checkpoint.hpp:11-50): 0 = snapshots in HBM
   (default), 1 = snapshots spilled to pinned host memory on a copy stream that overlaps the
   forward, brought back when the backward replays their segment.  Results are identical. */
int flume_set_checkpoint_spill(flume_ctx* ctx, int mode);
/* The file tier (NVMe; PAPER.md's offload): snapshots other than the last segment's go to an
   anonymous file in `dir` (D2H into pinned staging buffers on a copy stream, written by a
   worker thread; read back -- the next older one prefetched -- when the backward replays).
   Results identical to the other tiers.  flume_set_checkpoint_spill(ctx, 0 / 1) switches back. */
int flume_set_checkpoint_spill_dir(flume_ctx* ctx, const char* dir);
/* trajectory_chamfer nearest-neighbour search (losses.hpp:15-64): 0 = automatic (brute-force
   scan for small member x goal sets, a uniform-grid index above 2^24 pairs), 1 = always the
   scan, 2 = always the grid index.  Both return the reference's first-index minimum, so the
   loss and gradient bits do not depend on the mode. */
int flume_set_chamfer_mode(flume_ctx* ctx, int mode);
/* Particle sort between substeps: 1 (default) = incremental when the state came out of the
   previous substep on this context (only the blocks a particle entered, left or moved
   inside are re-sorted; the rest keep their order), 0 = always the full block counting
   sort.  Identical order, so identical results.  flume_sort_stats counts both kinds. */
int flume_set_incremental_sort(flume_ctx* ctx, int on);
int flume_sort_stats(const flume_ctx* ctx, long* incremental, long* full);
int flume_get_stream(flume_ctx* ctx, void** cuda_stream);
int flume_sync(flume_ctx* ctx);
int flume_last_timing(const flume_ctx* ctx, flume_timing* out);

/* ---- x-slab decomposition over several ranks ----
 * Rank r owns the 4-cell columns [sx0, sx1) along x (split by particle count at
 * upload); neighbours exchange two halo planes per scatter and migrating
 * particles, everything else is all-reduced.  Every call on a rank context is
 * collective: all ranks make the same calls in the same order, concurrently.
 * The results equal one rank's: particle states bit-identical, losses and
 * action gradients up to the order of their final sums.
 *   flume_group_create     n contexts in this process (one host thread per rank;
 *                          ranks may share a device), peer copies over NVLink
 *   flume_ctx_create_dist  one context per process (torchrun), NCCL; all ranks
 *                          pass the id rank 0 got from flume_dist_unique_id (or
 *                          flume_ipc_unique_id: CUDA IPC within one node) */
int flume_group_create(const flume_scene_desc* desc, int n_ranks, const int* devices, flume_ctx** out_ctxs);
int flume_dist_unique_id(unsigned char uid[128]);
/* group id for the CUDA-IPC transport instead of NCCL: the processes of one node (one or
 * several ranks per GPU) copy into each other's IPC-exported device inboxes (NVLink
 * between GPUs), ordered by interprocess events; pass it to flume_ctx_create_dist */
int flume_ipc_unique_id(unsigned char uid[128]);
int flume_ctx_create_dist(const flume_scene_desc* desc, int device, int rank, int n_ranks,
                          const unsigned char uid[128], flume_ctx** out);
int flume_slab_info(const flume_ctx* ctx, int* rank, int* n_ranks, int* sx0, int* sx1, long* n_active);
/* Migrating particles travel in fixed-size messages of `capacity` slots per neighbour
 * and substep (counts stay on the device: no host round trip per substep).  A call
 * whose migration exceeds it is re-run from its start with 4x the capacity (same
 * result); `retries` counts those re-runs.  Collective: every rank sets the same value. */
int flume_slab_set_migration_capacity(flume_ctx* ctx, int capacity);
int flume_slab_migration_stats(const flume_ctx* ctx, int* capacity, long* retries);
/* the column split every rank computes at upload: weights = active particles per
 * 4-cell x column, cuts[n_ranks + 1] (host-only, no device needed) */
int flume_slab_split(const double* col_weight, int n_cols, int n_ranks, int* cuts);

/* ---- instrumentation ----
 * flume_profile: time every kernel class with CUDA events on the context stream.
 * kernel classes: 0 p2g, 1 grid_update, 2 g2p, 3 sort+block lists, 4 g2p adjoint,
 * 5 grid adjoint, 6 p2g adjoint, 7 rigid (fwd+adj), 8 other, 9 slab halo / migration
 * exchanges (pack, transport, unpack) */
int flume_profile(flume_ctx* ctx, int enable);
int flume_kernel_times(flume_ctx* ctx, double* ms, long* counts, int n);
int flume_timer_mark(flume_ctx* ctx, int slot); /* slot 0..7: cudaEventRecord on the context stream */
int flume_timer_elapsed(flume_ctx* ctx, int a, int b, double* ms);

/* ---- state hand-off ---- */
int flume_state_upload(flume_ctx* ctx, const flume_state_view* view);
int flume_state_download(flume_ctx* ctx, flume_state_view* view);
/* the store as it is: cell keys, particle ids and active count (n entries each).  The slots
   are in the last sort's order, the keys those of the stored positions (after a substep they
   may no longer be sorted: the next substep sorts them) */
int flume_store_order(flume_ctx* ctx, unsigned* keys, unsigned* ids, long* n_active);
/* fp32 positions in store order (for the bit-exact key/order check) */
int flume_store_positions(flume_ctx* ctx, float* x);
/* the canonical (cell key, id) order of the current store as the next substep's sort
   produces it (incremental when possible): keys, ids and fp32 positions ([3][N], SoA) of the
   first n_keep slots in sorted order.  One-rank contexts. */
int flume_store_sorted(flume_ctx* ctx, unsigned* keys, unsigned* ids, float* x, long* n_active);

/* ---- hot path ---- */
int flume_substep(flume_ctx* ctx, const double action[6], int count);
int flume_stage_grid(flume_ctx* ctx, double* mass, double* vel); /* dense (i*ny+j)*nz+k order */
int flume_rollout_loss(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss, long window,
                       double* loss_out, double* per_segment);
/* rollout_loss with its final_state out-parameter (grad.hpp:15-41): the same loss, and the
   context's state becomes the state after the whole horizon (read it with
   flume_state_download) instead of staying at state0 */
int flume_rollout_loss_final(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss, long window,
                             double* loss_out, double* per_segment);
int flume_grad_trajectory(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss, long stride,
                          long window, double* action_grad, double* loss_out, double* full_loss,
                          double* per_segment, long* snapshots);
/* LossEvaluator::per_particle (losses.hpp:367-390) of the context's state: per particle id,
   the sum over the loss terms on its body of its unweighted distance (target_point,
   hold_initial, nearest point of the last trajectory_chamfer goal set); feeds
   flume_loss_desc.prev_losses of the next optimizer iterate.  Single-rank contexts. */
int flume_loss_per_particle(flume_ctx* ctx, const flume_loss_desc* loss, double* out);
int flume_adjoint_substep(flume_ctx* ctx, const double action[6], double* x_bar, double* v_bar, double* F_bar,
                          double* C_bar, double* eff_bars /* n_eff*12: t_bar[3], R_bar[9] */,
                          double* action_bar);

#ifdef __cplusplus
}
#endif

#endif /* FLUME_B200_H */
