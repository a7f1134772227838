/*
 * twg.h -- C ABI of the B200-native Time-Warped Grid hot path
 * (arXiv 1903.07441, "Dynamic Path Planning via Time-Warped Grids").
 *
 * The library (libtwg.so, built from paper_1903_07441_b200/csrc/) runs every
 * step of the planner's data-parallel hot path in hand-written sm_100a CUDA
 * kernels:
 *   a1-a3  time-warped obstacle rasterisation   twg_set_obstacles
 *   a4-a6  red-black Laplace relaxation + residual + convergence control
 *                                                twg_relax
 *   a7-a9  descent walk + rubber band + next waypoint
 *                                                twg_extract_path
 *   all    one planning tick (Algorithm 1)       twg_plan_step
 *
 * Citations: "P:n" = PAPER.md line n (Eq./Alg. named), "S:n" = SPEC.md line n,
 * "C<k>" = the reading recorded in DESIGN.md "Readings of the paper".
 *
 * Conventions (apply to every call):
 *  - Ownership: the caller owns every array passed in or out.  Inputs are
 *    copied during the call; no caller pointer is retained.  The context owns
 *    its device buffers.
 *  - Pointers marked "host or device" are classified with
 *    cudaPointerGetAttributes; device pointers must live on the context's
 *    device.  All other pointers are host pointers.
 *  - Stream order: all device work is enqueued on the context stream (the one
 *    passed to twg_create, e.g. torch.cuda.current_stream().cuda_stream).
 *    A call that returns host data synchronises that stream before returning.
 *  - Errors: a negative status means the call wrote no outputs (except where
 *    stated); the message is available from twg_last_error.  Positive status
 *    values are warnings; outputs are valid.  Nothing throws across the ABI.
 *  - A context is single-owner; distinct contexts may be used
 *    concurrently from different threads.
 *  - Grid coordinates: cell (x, y), x = column in [0, width), y = row in
 *    [0, height), row-major; world point p belongs to cell
 *    floor((p - origin) / cell_size).
 *  - Field encoding on the device ("raw u", used by twg_get_field(raw) and
 *    twg_set_field): u = 1 - phi stored as fp32 (C3) with the sign bit as the
 *    free/fixed flag: a free cell holding u >= 0 is stored as -u (sign bit
 *    set); a fixed cell is stored non-negative: obstacle +0.0 (phi = 1),
 *    goal +1.0 (phi = 0).  Any other non-negative value is a fixed Dirichlet
 *    cell with that u (test data, pin P8).  Every |u| must lie in [0, 1]
 *    (the range of u = 1 - phi; the index kernel orders |u| on its bits).  Outside the grid u = +0.0
 *    (obstacle, C4).
 */
#ifndef TWG_H
#define TWG_H

#include <stdint.h>

#ifdef __cplusplus
#define TWG_API extern "C" __attribute__((visibility("default")))
#else
#define TWG_API __attribute__((visibility("default")))
#endif

typedef struct twg_ctx twg_ctx; /* opaque; owns the device state of `batch` scenarios */
typedef int32_t twg_status;

enum {
    TWG_OK = 0,
    TWG_W_GOAL_SWALLOWED = 1,      /* a footprint covered the goal cell; the goal was kept */
    TWG_W_TRUNCATED = 2,           /* output longer than its capacity; truncated */
    TWG_W_SINGULAR_INNOVATION = 3, /* a matched track's H P H^T + R was not positive definite;
                                      the track kept its prediction */
    TWG_E_INVALID_ARG = -1,
    TWG_E_OUT_OF_BOUNDS = -2,      /* goal or robot cell outside the grid */
    TWG_E_OVERLAPPING_CLASSES = -3,/* goal on a static wall */
    TWG_E_INVALID_START = -4,      /* robot cell on a static wall */
    TWG_E_NO_PATH = -5,            /* walk entered an obstacle or exceeded max_len (C9) */
    TWG_E_CUDA = -6,
    TWG_E_NCCL = -7,
    TWG_E_NO_MEMORY = -8
};

/* Grid of `batch` independent scenarios of width x height cells of
 * cell_size metres (0.1 m), cell (0,0)'s corner at (origin_x,
 * origin_y).
 * Row slabs come in two forms:
 *  - sharded contexts (twg_create with an NCCL communicator, or
 *    twg_create_group): the desc is the GLOBAL grid (batch 1, row_offset 0,
 *    ghost_rows 0) and exchange_every = k >= 1 sweeps between ghost
 *    exchanges; the library gives slab r of n the owned global rows
 *    [r0, r1) = [r H/n, (r + 1) H/n) (near-equal split) plus G = 2k ghost rows
 *    per side, exchanges them inside twg_relax and max-reduces the residual
 *    across slabs on the device (twg_slab_info reports the geometry);
 *  - manual slabs (no communicator): row_offset = global index of local row
 *    0, so the red/black colour is the parity of (x + row_offset + y) (C1);
 *    ghost_rows = G rows at the top and at the bottom of the local grid that
 *    the caller keeps as copies of the neighbouring slabs (owned rows are
 *    [G, height - G)).
 * With G > 0 the residual of twg_relax covers the owned rows only, the goal
 * and the robot may lie outside the local grid (their cells are then simply
 * absent) and twg_plan_step is not available; twg_extract_path works on
 * sharded contexts (the walk is handed over between the slabs and every slab
 * returns the whole path in global cells, see twg_extract_path) but not on
 * manual slabs (hand the walk over with twg_walk_from).  Single-GPU contexts
 * pass 0 for row_offset, ghost_rows and exchange_every. */
typedef struct {
    int32_t width, height, batch, row_offset;
    int32_t ghost_rows, exchange_every;
    double cell_size, origin_x, origin_y;
} twg_grid_desc;

/* Robot pose and speed: metres, metres, radians (heading theta of Eq. 14,
 * P:462), m/s ("velocity of the robot"). */
typedef struct {
    double x, y, theta, speed;
} twg_robot;

/* Kalman track of one moving obstacle: state (x, y, vx, vy) in
 * m and m/s and its 4x4 covariance P, row-major (Eq. 10). */
typedef struct {
    double x[4];
    double P[16];
} twg_track;

/* Time-warp / predict configuration (defaults in brackets):
 *   dt [0.1 s] Kalman step; Q [1e-3 diag(dt^4/4, dt^4/4, dt^2, dt^2), S:307]
 *   process noise, row-major; warp_spacing [1.0 m] width of one warp ring
 *   (C17); eps_v [0.05 m/s] obstacle-speed floor of Eq. 16 (C18);
 *   safety_radius [0.5 m] (C20); horizon_max [20] clamp of j (C18);
 *   horizon_mode [0]: 0 = Eq. 16, j = round(v t), v = speed ratio (C18);
 *     1 = time the robot needs to reach ring t, j = round(t w / (speed_r dt))
 *     (north_star wording; C26);
 *   footprint_mode [0]: 0 = covariance after the j predicts (C19);
 *     1 = the track's own posterior covariance P_k|k (C27). */
typedef struct {
    double dt;
    double Q[16];
    double warp_spacing;
    double eps_v;
    double safety_radius;
    int32_t horizon_max;
    int32_t horizon_mode;
    int32_t footprint_mode;
    int32_t reserved;
} twg_warp_cfg;

/* Relaxation control (rows a4-a6):
 *   max_sweeps [100, Alg. 1 P:694]; check_every [max_sweeps]: the residual
 *   max|du| of sweep s is evaluated when s % check_every == 0 or s ==
 *   max_sweeps (C5); stop early when it is < tol (tol <= 0: fixed budget,
 *   C6); warm_start [1]: used by twg_plan_step's encode (C7);
 *   temporal_depth [0 = auto = 6]: sweeps fused per tile load (T, 1..8);
 *   with both temporal_depth and rows_per_warp 0, a grid of at most 40960
 *   cells is solved by one CTA per scenario in shared memory (all sweeps,
 *   the residual and the stop rule in one launch; same result);
 *   rows_per_warp [0 = auto, load model of DESIGN.md]: rows of the strip one
 *   warp owns;
 *   sync_every [64]: convergence flags are read back every sync_every
 *   checks when tol > 0;
 *   mode [0]: 0 = red-black Gauss-Seidel (Eq. 2, the hot path);
 *   1 = Jacobi (Eq. 1: every free cell from the previous iterate);
 *   2 = lexicographic Gauss-Seidel (Eq. 2 literally: row-major order, W and N
 *   from this sweep; not on row slabs); modes 1, 2 ignore temporal_depth and
 *   rows_per_warp. */
typedef struct {
    int32_t max_sweeps, check_every, warm_start, temporal_depth;
    float tol;
    int32_t rows_per_warp, sync_every, mode;
} twg_relax_cfg;

/* Path output control (rows a7-a9):
 *   iterations [50] rubber-band iterations (C10); max_len: walk cells
 *   capacity (NoPath beyond); max_smooth: smoothed points capacity;
 *   step [0.25 cell] candidate offset (C12); k_t [1.0] tension constant (C11). */
typedef struct {
    int32_t iterations, max_len, max_smooth, reserved;
    float step, k_t;
} twg_band_cfg;

/* Tracker configuration (row f1, the step before a1 in Alg. 1's Map Update,
 * P:680-688):
 *   sigma_z [0.05 m]: measurement noise, R = sigma_z^2 I;
 *   gate [0.5 m]: a (track, detection) pair is a candidate iff the squared
 *     distance from the predicted position is <= gate^2;
 *   spawn_var_pos [0.25 m^2], spawn_var_vel [1.0 (m/s)^2]: covariance
 *     diagonal of a track spawned from an unmatched detection;
 *   prune_after [10]: tracks with missed > prune_after are removed;
 *   max_tracks [0 = no limit]: tracks kept per scenario after the tick. */
typedef struct {
    double sigma_z, gate, spawn_var_pos, spawn_var_vel;
    int32_t prune_after, max_tracks;
} twg_tracker_cfg;

/* n / n_tracks value selecting the context's resident tracker table. */
#define TWG_RESIDENT_TRACKS (-1)

/* Closed-loop simulator (row f2; C31-C36), defaults in brackets:
 *   dt [0.1 s]; robot_radius, obstacle_radius [0.25 m]; goal_radius [0.3 m];
 *   turn_distance [0.5 m] obstacles turn away from walls / obstacles this
 *   far ahead; heading_sigma [0.02 rad] obstacle heading jitter;
 *   det_sigma [0.05 m] detection noise; turn_max [9 deg = 90 deg/s
 *   at dt 0.1] robot turn per tick; seed of the counter-based
 *   generator (C31); max_ticks [1000] trial time limit; init_tol [1e-6],
 *   init_max_sweeps [1e6]: the tick-0 field is relaxed to this residual
 *   (Alg. 1 "Initialize ... harmonic potential values"; C36). */
typedef struct {
    double dt, robot_radius, obstacle_radius, goal_radius, turn_distance, heading_sigma, det_sigma, turn_max;
    uint64_t seed;
    int32_t max_ticks, init_max_sweeps;
    float init_tol;
    int32_t reserved;
} twg_sim_cfg;

/* State of one trial. status: 0 running, 1 success (robot centre within
 * goal_radius of the goal cell centre), 2 collision (robot centre outside
 * the grid, a static wall cell centre within robot_radius, or an obstacle
 * closer than robot_radius + obstacle_radius), 3 timeout,
 * 4 idle (never reset).  (hx, hy): unit heading; length: distance
 * travelled (m). */
typedef struct {
    double x, y, hx, hy, speed, length;
    int32_t ticks, status;
} twg_sim_trial;

/* Result of one planning tick.  next_x/next_y: next waypoint in cell units
 * (cell (i, k) has centre (i + 0.5, k + 0.5)) (Alg. 1). */
typedef struct {
    twg_status status;      /* worst status of the tick (errors < 0 < warnings) */
    int32_t sweeps;         /* sweeps performed */
    int32_t n_cells;        /* descent-walk cells (0 on NoPath) */
    int32_t n_smooth;       /* smoothed + resampled points (may exceed max_smooth: truncated) */
    float residual;         /* max |du| of the last sweep (C5) */
    float next_x, next_y;   /* next waypoint (cell units) */
    int32_t walk_status;    /* TWG_OK or TWG_E_NO_PATH */
} twg_plan_result;

/* Create a context for `desc->batch` scenarios on CUDA device `device`,
 * enqueuing on `cuda_stream` (a cudaStream_t; NULL = the legacy default
 * stream).  Allocates 2 ping-pong fields of height x pitch fp32 per scenario
 * (pitch = width rounded up to 32) plus a uint8 static mask.  Every field
 * starts as all-free cold (u = 0.5) with no goal.
 * nccl_comm: NULL = single GPU (or a manual slab); else an ncclComm_t (from
 * twg_nccl_comm_init, or any communicator of the same libnccl.so.2, e.g.
 * torch's ProcessGroupNCCL._comm_ptr()) whose rank r of n makes this context
 * slab r of the global grid `desc` (row slabs; see
 * twg_grid_desc).  Every rank must then call twg_relax with the same
 * configuration: the ghost rows are exchanged with ncclSend / ncclRecv every
 * exchange_every sweeps on a high-priority stream, overlapped with the
 * interior tiles, and the residual is max-all-reduced (ncclAllReduce) before
 * the stop rule is evaluated on the device.  The communicator is borrowed: it
 * must outlive the context.
 * Errors: INVALID_ARG (sizes <= 0, cell_size <= 0, batch > 65535; slabs: batch
 * != 1, exchange_every < 1, a slab thinner than 2 exchange_every rows), CUDA,
 * NCCL, NO_MEMORY. */
TWG_API twg_status twg_create(const twg_grid_desc* desc, int32_t device, void* cuda_stream, void* nccl_comm,
                              twg_ctx** out);

/* nslabs (1..16) row-slab contexts of the global grid `desc` on one device,
 * out[nslabs] in slab order (a local group: the row-slab decomposition of
 * twg_create with a communicator, with ghost rows exchanged by device copies
 * instead of NCCL).  twg_relax on any member relaxes the whole
 * group (sweeps_done / residual are the group's).  Destroy every member;
 * destroying one detaches the others (they then act as manual slabs).
 * Errors as twg_create. */
TWG_API twg_status twg_create_group(const twg_grid_desc* desc, int32_t nslabs, int32_t device, void* cuda_stream,
                                    twg_ctx** out);

/* Slab geometry of ctx: out8 = {rank, nranks, r0, r1 (owned global rows
 * [r0, r1)), row_offset (global row of local row 0), ghost_rows,
 * exchange_every, local height}.  Unsharded: {0, 1, ...}. */
TWG_API twg_status twg_slab_info(const twg_ctx* ctx, int32_t* out8);

/* NCCL communicator helpers for sharded contexts (the library resolves NCCL
 * at run time from the libnccl.so.2 the process has loaded, e.g. torch's).
 * twg_nccl_unique_id: ncclGetUniqueId into out (bytes >= 128; broadcast it to
 * every rank, e.g. with torch.distributed); twg_nccl_comm_init:
 * ncclCommInitRank on `device` (collective over the nranks ranks);
 * twg_nccl_comm_destroy: ncclCommDestroy.  Errors: INVALID_ARG, NCCL, CUDA. */
TWG_API twg_status twg_nccl_unique_id(void* out, int32_t bytes);
TWG_API twg_status twg_nccl_comm_init(int32_t nranks, const void* id, int32_t rank, int32_t device, void** comm);
TWG_API twg_status twg_nccl_comm_destroy(void* comm);

/* Release all device memory of the context.  NULL is a no-op. */
TWG_API twg_status twg_destroy(twg_ctx* ctx);

/* Static wall mask of scenario b (b = -1: every scenario), height x width
 * uint8 row-major, non-zero = wall ("phi(x,y) = 1"; P:586 red lines).
 * Sharded contexts take the GLOBAL mask and keep their local rows (rows
 * outside the global grid are walls, C4).
 * Host or device pointer.  The next twg_set_obstacles re-encodes cold. */
TWG_API twg_status twg_set_static(twg_ctx* ctx, int32_t b, const uint8_t* occ);

/* Rows a1-a3 for scenario b (Alg. 1 Map Update):
 *   a1 warp radius of each track from its current estimate (Eq. 15 closed
 *      form, C16; warp number t, C17);
 *   a2 horizon j = clamp(round(v t)) (Eq. 16, C18) and j Kalman predicts
 *      (Eqs. 9-10) giving the footprint R^2 (C19, C20);
 *   a3 field encode: cells whose centre lies within R of a predicted
 *      position become obstacles, static walls stay obstacles, the goal cell
 *      is the goal, the robot's cell stays free (C22).
 * Sharded contexts take the goal in global cells.
 * warm = 0: every free cell restarts at 0.5 ("cleared");
 * warm = 1: every free cell keeps the value it holds, including cells fixed
 * in the previous call and free now (a released obstacle keeps u = 0), except
 * a released goal, which restarts at u = 0 (a free cell at u = 1 would be a
 * spurious maximum) ("the values evolve slowly"; C7).
 * tracks: n entries, host or device pointer (n may be 0); they also replace
 * the scenario's resident tracker table (missed counters 0).  tracks = NULL
 * with n = TWG_RESIDENT_TRACKS: use the resident table as left by
 * twg_track_update (row f1).
 * Returns OK, W_GOAL_SWALLOWED, or OUT_OF_BOUNDS / OVERLAPPING_CLASSES /
 * INVALID_START / INVALID_ARG (validated before any device work). */
TWG_API twg_status twg_set_obstacles(twg_ctx* ctx, int32_t b, const twg_robot* robot,
                                     int32_t goal_x, int32_t goal_y,
                                     const twg_track* tracks, int32_t n,
                                     const twg_warp_cfg* cfg, int32_t warm);

/* Rows a4-a6 for every scenario: red-black Gauss-Seidel relaxation of
 * Eq. 2 realised as red pass then black pass per sweep (C1),
 * each free cell u <- 0.25 ((E + W) + (N + S)) (C2), with the residual
 * and stop rule of cfg.  sweeps_done[batch] and residual[batch] are host
 * arrays; if both are NULL and cfg->tol <= 0 the call does not synchronise.
 * Errors: INVALID_ARG (max_sweeps < 0, check_every < 0), CUDA. */
TWG_API twg_status twg_relax(twg_ctx* ctx, const twg_relax_cfg* cfg, int32_t* sweeps_done, float* residual);

/* Rows a7-a9 for scenario b on the current field:
 *   a7 descent walk from the robot cell of the last twg_set_obstacles along
 *      the implicit index matrix of Eq. 3 (argmax u, order +x, -x, +y, -y,
 *      first maximum wins, C8), into cells_xy (max_len (x, y) int32 pairs);
 *   a8 rubber band (Eqs. 4-6, C10-C14) of the cell-centre waypoints, then
 *      resampling (C15) into smooth_xy (max_smooth (x, y) float pairs);
 *   a9 next waypoint into next_xy[2] (cell units).
 * Host arrays; any output pointer may be NULL.  Returns OK, W_TRUNCATED or
 * NO_PATH (then *n_cells = *n_smooth = 0 and next_xy = robot cell centre).
 * Sharded contexts (b = 0; every slab of the group calls it, NCCL ranks
 * collectively): the walk runs on the slab owning the current cell and is
 * handed to the neighbouring slab when it steps into a ghost row (ncclBroadcast
 * of the walker state); the band and the resampling run on the rows of the
 * global grid within I step sqrt(2) + 3 of the path, assembled from the slabs
 * (SURVEY 8(e)); cells, smooth points and next waypoint are in global
 * coordinates and identical on every slab. */
TWG_API twg_status twg_extract_path(twg_ctx* ctx, int32_t b, const twg_band_cfg* cfg,
                                    int32_t* cells_xy, int32_t* n_cells,
                                    float* smooth_xy, int32_t* n_smooth, float* next_xy);

/* One planning tick (Algorithm 1) = twg_set_obstacles (warm =
 * relax->warm_start) + twg_relax + twg_extract_path.
 * b >= 0: scenario b; robot, goal_xy[2], tracks[n_tracks[0]], out[1],
 *   cells_xy[2 max_len], smooth_xy[2 max_smooth].
 * b = -1: every scenario; robot[batch], goal_xy[2 batch], tracks = the
 *   concatenation of n_tracks[0..batch) tracks, out[batch],
 *   cells_xy[batch][2 max_len], smooth_xy[batch][2 max_smooth].
 * tracks may be host or device; every other pointer is host (cells_xy,
 * smooth_xy may be NULL; for b >= 0 only the entries produced are written).  tracks = NULL and n_tracks = NULL: every
 * scenario uses its resident tracker table (row f1).
 * Returns the worst per-scenario status. */
TWG_API twg_status twg_plan_step(twg_ctx* ctx, int32_t b, const twg_robot* robot, const int32_t* goal_xy,
                                 const twg_track* tracks, const int32_t* n_tracks,
                                 const twg_warp_cfg* warp, const twg_relax_cfg* relax,
                                 const twg_band_cfg* band, twg_plan_result* out,
                                 int32_t* cells_xy, float* smooth_xy);

/* Copy scenario b's current field (height x width fp32, row-major, no
 * pitch) to `out` (host or device).  mode 0: raw u (header encoding);
 * 1: |u| (u-space magnitudes); 2: phi = 1 - |u|. */
TWG_API twg_status twg_get_field(twg_ctx* ctx, int32_t b, float* out, int32_t mode);

/* Replace scenario b's current field by `raw` (height x width, raw u
 * encoding, host or device) -- warm start / checkpoint restore / test data. */
TWG_API twg_status twg_set_field(twg_ctx* ctx, int32_t b, const float* raw);

/* Per-track results of the last twg_set_obstacles on scenario b (rows a1-a2,
 * for parity tests): t[n] warp numbers, j[n] horizons, pred[3 n] =
 * (x_pred, y_pred, R^2).  n must equal the track count of that call. */
TWG_API twg_status twg_get_warp(twg_ctx* ctx, int32_t b, int32_t n, int32_t* t, int32_t* j, double* pred);

/* Row f1: one tracker tick on the resident track table of scenario b
 * (b = -1: every scenario) -- Alg. 1 P:680-688 "Read ... Detect ...
 * Estimate":
 *   1. every track predicted one step (Eqs. 9-10; dt, Q of `warp`);
 *   2. greedy gated association: repeatedly the globally closest free
 *      (track, detection) pair within the gate, ties to the lower track
 *      then the lower detection index (C29);
 *   3. matched tracks: Kalman update Eqs. 11-13 with
 *      H = [I2 0], R = sigma_z^2 I, then P <- (P + P^T) / 2
 *      (C28), missed = 0; unmatched tracks keep the prediction, missed + 1;
 *   4. tracks with missed > prune_after removed, order kept;
 *   5. one track per unmatched detection appended in detection order,
 *      x = (z, 0, 0), P = diag(var_pos, var_pos, var_vel, var_vel);
 *   6. at most max_tracks kept (survivors first; W_TRUNCATED).
 * det_xy: (x, y) metres, host or device; b >= 0: n_det[0] detections;
 * b = -1: the concatenation of n_det[0..batch) (host array) detections.
 * n_tracks (host, may be NULL): track count per scenario after the tick.
 * Synchronises.  Returns OK, W_TRUNCATED, W_SINGULAR_INNOVATION or
 * INVALID_ARG (sigma_z, gate, variances < 0, prune_after < 0). */
TWG_API twg_status twg_track_update(twg_ctx* ctx, int32_t b, const double* det_xy, const int32_t* n_det,
                                    const twg_warp_cfg* warp, const twg_tracker_cfg* cfg, int32_t* n_tracks);

/* Copy scenario b's resident tracker table: up to cap tracks into out and
 * their missed counters into missed (host or device; either may be NULL);
 * *n = the table's track count. */
TWG_API twg_status twg_get_tracks(twg_ctx* ctx, int32_t b, twg_track* out, int32_t* missed, int32_t cap, int32_t* n);

/* Row f2: start trial b of the closed-loop simulator.  robot: start pose
 * and constant speed (the robot never stops); goal cell;
 * obstacles[n][4] = (x, y, vx, vy) true states (host), constant speed
 * sqrt(vx^2 + vy^2).  Clears b's tracker table, encodes the static map and
 * goal cold and relaxes that field to cfg->init_tol (C36), and produces the
 * tick-0 detections.  Errors: INVALID_ARG, OUT_OF_BOUNDS, INVALID_START,
 * OVERLAPPING_CLASSES (as twg_set_obstacles), CUDA. */
TWG_API twg_status twg_sim_reset(twg_ctx* ctx, int32_t b, const twg_robot* robot, int32_t goal_x, int32_t goal_y,
                                 const double* obstacles, int32_t n, const twg_sim_cfg* cfg);

/* Row f2: one tick of every running trial -- Algorithm 1 closed loop
 * (P:674-709): tracker tick on the current detections (row f1), Map Update
 * from the resident tracks (a1-a3, robot heading theta = atan2(hy, hx)),
 * relaxation (a4-a6), path (a7-a9), then the simulator step (robot toward
 * the next waypoint, or straight on when no path exists; obstacles
 * move; status) and the next tick's detections.  out[batch] (host, may be
 * NULL) receives every trial's state, *running the number still running.
 * Returns the worst planner status of the tick (warnings >= 0) or an
 * error. */
TWG_API twg_status twg_sim_tick(twg_ctx* ctx, const twg_sim_cfg* cfg, const twg_warp_cfg* warp,
                                const twg_relax_cfg* relax, const twg_band_cfg* band, const twg_tracker_cfg* tracker,
                                twg_sim_trial* out, int32_t* running);

/* Row f2: trial b's turning-angle histogram, hist[36] (bin k: per-tick
 * heading change in [5k, 5k + 5) degrees), host. */
TWG_API twg_status twg_sim_histogram(twg_ctx* ctx, int32_t b, int32_t* hist);

/* Descent walk from local cell (x, y) of scenario b on the current field, for
 * row slabs (the walker is handed from slab to slab).  Follows
 * Eq. 3 (argmax u over the in-grid 4-neighbours, order +x, -x, +y, -y, C8)
 * from (x, y), appending every visited cell (local coordinates, the start
 * included) to cells_xy (host, max_cells pairs), until: the goal
 * (*code = 0); the next cell lies in a ghost row, i.e. belongs to the
 * neighbouring slab (*code = 1 above, 2 below; next_xy = that cell, not
 * appended); an obstacle, no neighbour, or more than max_cells cells
 * (*code = TWG_E_NO_PATH).  The ghost rows must hold the neighbours' current
 * rows (exchange them after the last relaxation).  On an unsharded grid the
 * walk never hands over.  Correctness path, one thread. */
TWG_API twg_status twg_walk_from(twg_ctx* ctx, int32_t b, int32_t x, int32_t y, int32_t max_cells,
                                 int32_t* cells_xy, int32_t* n_cells, int32_t* code, int32_t* next_xy);

/* Full-grid index matrix M_idx of scenario b's current field (Eq. 3,
 * P:228-233; Alg. 1): out[height x width] uint8
 * row-major (host or device): 0..3 = step to the in-grid neighbour with the
 * largest u, order +x, -x, +y, -y, first maximum wins (C8); 4 goal;
 * 5 obstacle; 6 no in-grid neighbour (1 x 1 grid).  Cells on a slab's
 * ghost rows use the local grid only.  Errors: INVALID_ARG, CUDA. */
TWG_API twg_status twg_index_matrix(twg_ctx* ctx, int32_t b, uint8_t* out);

/* Per-cell rubber band on the index matrix (Alg. 1 P:701-704 "for each cell
 * in the index matrix in parallel: calculate tension force T and potential
 * force F via Eq. 6; update the index matrix with the position of the
 * neighbor with the minimum resultant force (Eqs. 4-5)", then P:705
 * "generate the current path based on the optimized index matrix"; SURVEY
 * 8(f) f3; reading C37): M_idx of Eq. 3 for scenario b's current field, then
 * cfg->iterations iterations (cells with (x + y) even, then odd) in which
 * every free cell c picks, among its in-grid non-obstacle 4-neighbours n with
 * u > 1e-9, the successor minimising |R|^2, R = -F d + k_t (c - n) +
 * k_t (M(n) - n), F = 1/u(n) - 1/u(c) (C13), the current successor kept on
 * ties, the others in the order +x, -x, +y, -y; then the walk along the
 * optimised matrix from the robot cell.  out[height x width] (host or device,
 * may be NULL): the optimised matrix (codes of twg_index_matrix); cells_xy
 * (host, max_len (x, y) pairs, may be NULL), *n_cells: the walk.  Not on row
 * slabs.  Returns OK or NO_PATH (the walk met an obstacle, a successor-less
 * cell or exceeded max_len; *n_cells = 0); INVALID_ARG, CUDA. */
TWG_API twg_status twg_band_index(twg_ctx* ctx, int32_t b, const twg_band_cfg* cfg, uint8_t* out, int32_t* cells_xy,
                                  int32_t* n_cells);

/* Per-cell warp number (the paper's kernel 1, "calculate the warp
 * of each cell"; the numbered ellipses of P:438-456):
 * out[height x width] int32 row-major (host or device), t = max(1,
 * ceil(r_x / warp_spacing)) of an obstacle at the cell centre (C16, C17)
 * for the robot pose `robot` on this context's grid geometry (origin,
 * cell_size; a slab's local rows).  Errors: INVALID_ARG
 * (warp_spacing <= 0), CUDA. */
TWG_API twg_status twg_warp_map(twg_ctx* ctx, const twg_robot* robot, double warp_spacing, int32_t* out);

/* Device pointer and pitch (floats) of scenario b's current field buffer
 * (valid until the next call on ctx). */
TWG_API twg_status twg_field_ptr(twg_ctx* ctx, int32_t b, void** dev_ptr, int64_t* pitch);

/* Kernel-level accounting for bench.py: total kernel launches enqueued by
 * this context since creation, and, while profiling is enabled, CUDA-event
 * time and launch count of the relaxation tile kernel (the dominant kernel),
 * plus the lattice updates those launches performed. */
TWG_API int64_t twg_kernel_launches(const twg_ctx* ctx);
TWG_API twg_status twg_profile(twg_ctx* ctx, int32_t enable);
TWG_API twg_status twg_profile_read(twg_ctx* ctx, double* relax_ms, int64_t* relax_launches, int64_t* cell_sweeps);

/* Cycle accounting of the last descent walk of scenario b (performance
 * debugging): out4 = {staging, chase, flush} in kilo-cycles of the walking
 * thread, and the number of windows staged. */
TWG_API twg_status twg_debug_walk(twg_ctx* ctx, int32_t b, int32_t* out4);

/* Message of the last error on ctx ("" if none); ctx NULL: last twg_create error. */
TWG_API const char* twg_last_error(const twg_ctx* ctx);

#endif /* TWG_H */
