/*
 * twg_oracle.c -- plain, slow CPU oracle of the Time-Warped Grid hot path
 * (arXiv 1903.07441).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1903_07441_b200/) never includes, links or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "C<k>" = the reading recorded in DESIGN.md "Readings of the paper".
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared (no FMA
 * contraction, no FTZ/DAZ), so every float/double expression below is the
 * IEEE operation sequence written in the source, evaluated left to right.
 *
 * Representation: the oracle keeps its own uint8 class grid
 * (ORC_FREE / ORC_OBSTACLE / ORC_GOAL) and stores the field as
 * u = 1 - phi (C3), so goal u = 1, obstacle u = 0, free init 0.5.
 *
 * Parity-pinned functions: see the header of each function; the pins live in
 * tests/test_oracle_pins*.py (P1-P26).  Parity unpinned (defined only by the
 * algorithm as written here): the exact smoothed path on general scenes
 * (orc_band: one hand-computed step and its properties are pinned) and the
 * warm-start trajectory over many ticks (the warm initialisation itself and
 * the next-waypoint choice are pinned by hand, P25-P26).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_FREE = 0, ORC_OBSTACLE = 1, ORC_GOAL = 2 };
enum { ORC_OK = 0, ORC_W_GOAL_SWALLOWED = 1, ORC_E_INVALID_ARG = -1, ORC_E_OUT_OF_BOUNDS = -2,
       ORC_E_OVERLAPPING = -3, ORC_E_INVALID_START = -4, ORC_E_NO_PATH = -5 };

/* ------------------------------------------------------------------------ */
/* O1  time-warp radius and warp number  (Eqs. 14-15; C16, C17)  */
/* ------------------------------------------------------------------------ */

/* Eq. 15 is implicit because (x_c, y_c) depend on r_x.
 * With a = c dx + s dy, b = s dx - c dy (dx = x_obj - x_r): the rotated
 * offsets from the centre are a - 0.9 r and b, so Eq. 15 squared reads
 *   r^2 = (a - 0.9 r)^2 + 16 b^2  <=>  0.19 r^2 + 1.8 a r - (a^2 + 16 b^2) = 0,
 * whose unique non-negative root is (C16)
 *   r = (sqrt(4 a^2 + 12.16 b^2) - 1.8 a) / 0.38.                          */
double orc_warp_radius(double xr, double yr, double c, double s, double xo, double yo)
{
    double dx = xo - xr;
    double dy = yo - yr;
    double a = c * dx + s * dy;
    double b = s * dx - c * dy;
    return (sqrt(4.0 * a * a + 12.16 * b * b) - 1.8 * a) / 0.38;
}

/* Warp number t = max(1, ceil(r_x / w)) ("label the obstacle with
 * the corresponding warp number"; C17). */
int32_t orc_warp_number(double rx, double w)
{
    double t = ceil(rx / w);
    if (t < 1.0) t = 1.0;
    return (int32_t)t;
}

/* ------------------------------------------------------------------------ */
/* O2  horizon j and j-step Kalman predict  (Eqs. 9-10, 16-17)   */
/* ------------------------------------------------------------------------ */

/* Eq. 16: Time-Warp = v t, v = ratio of robot speed to obstacle
 * speed (C18): v = speed_r / max(|v_hat|, eps_v), j = clamp(round(v t), 0,
 * horizon_max), round = half away from zero (llround, C25). */
int32_t orc_horizon(int32_t t, double speed_r, double vx, double vy, double eps_v, int32_t hmax)
{
    double so = sqrt(vx * vx + vy * vy);
    if (so < eps_v) so = eps_v;
    double v = speed_r / so;
    long long j = llround(v * (double)t);
    if (j < 0) j = 0;
    if (j > hmax) j = hmax;
    return (int32_t)j;
}

/* Alternative horizon reading (north_star "the time the robot needs to reach that
 * grid ring"): ring t lies ~ t w metres away, reached after t w / speed_r seconds, i.e.
 * j = clamp(round(t w / (speed_r dt)), 0, horizon_max) Kalman steps (speed_r <= 0: horizon_max). */
int32_t orc_horizon_ring(int32_t t, double w, double speed_r, double dt, int32_t hmax)
{
    if (!(speed_r > 0.0)) return hmax;
    double steps = ((double)t * w) / (speed_r * dt);
    if (!(steps < 4.0e18)) return hmax;
    long long j = llround(steps);
    if (j < 0) j = 0;
    if (j > hmax) j = hmax;
    return (int32_t)j;
}

/* A of P:548-553: constant velocity, dt in the (0,2) and (1,3) slots. */
static void orc_A(double dt, double A[16])
{
    memset(A, 0, 16 * sizeof(double));
    A[0] = 1.0; A[5] = 1.0; A[10] = 1.0; A[15] = 1.0;
    A[0 * 4 + 2] = dt;
    A[1 * 4 + 3] = dt;
}

/* j applications of Eq. 9 (x <- A x) and Eq. 10 (P <- A P A^T + Q,
 * P:376), B = 0.  Dense 4x4 products, k ascending, separate * and +. */
void orc_predict(const double* x, const double* P, const double* Q, double dt, int32_t j,
                 double* xo, double* Po)
{
    double A[16], xc[4], Pc[16], AP[16], xn[4];
    orc_A(dt, A);
    memcpy(xc, x, sizeof xc);
    memcpy(Pc, P, sizeof Pc);
    for (int32_t step = 0; step < j; ++step) {
        for (int r = 0; r < 4; ++r) {
            double acc = 0.0;
            for (int k = 0; k < 4; ++k) acc = acc + A[r * 4 + k] * xc[k];
            xn[r] = acc;
        }
        memcpy(xc, xn, sizeof xc);
        for (int r = 0; r < 4; ++r)
            for (int col = 0; col < 4; ++col) {
                double acc = 0.0;
                for (int k = 0; k < 4; ++k) acc = acc + A[r * 4 + k] * Pc[k * 4 + col];
                AP[r * 4 + col] = acc;
            }
        for (int r = 0; r < 4; ++r)
            for (int col = 0; col < 4; ++col) {
                double acc = 0.0;
                for (int k = 0; k < 4; ++k) acc = acc + AP[r * 4 + k] * A[col * 4 + k];
                Pc[r * 4 + col] = acc + Q[r * 4 + col];
            }
    }
    memcpy(xo, xc, sizeof xc);
    memcpy(Po, Pc, sizeof Pc);
}

/* Footprint radius^2 (P:492-505 Gaussian "based on the calculated
 * uncertainty ... and a desired safety distance"; C19, C20):
 * sigma^2 = (P00 + P11) / 2; exp(-d^2 / (2 sigma^2)) >= 1/2  <=>
 * d^2 <= 2 ln 2 sigma^2; union with the safety disk d <= r_s. */
double orc_footprint_r2(const double* P, double rs)
{
    double sig2 = (P[0] + P[5]) * 0.5;
    double g = 1.3862943611198906 * sig2; /* 2 ln 2 */
    double s2 = rs * rs;
    return g > s2 ? g : s2;
}

/* ------------------------------------------------------------------------ */
/* O3  class grid: static walls, time-warped stamps, goal, robot exemption  */
/* (Alg. 1; C20-C22)                        */
/* ------------------------------------------------------------------------ */

/* tracks: n x 20 doubles (x[4], P[16] row-major).  Outputs the class grid
 * (row-major H x W), and per track t, j and (x_pred, y_pred, R^2).
 * Membership of cell (i, k): (ox + (i + 0.5) cs - xp)^2 + (oy + (k + 0.5) cs
 * - yp)^2 <= R^2 in double.  The loop box is a superset of the disk (pin P4
 * checks it against the all-cells loop, orc_stamp_bruteforce). */
static void orc_stamp_one(int32_t W, int32_t H, double cs, double ox, double oy,
                          double xp, double yp, double R2, uint8_t* stamp, int32_t box)
{
    int32_t i0 = 0, i1 = W - 1, k0 = 0, k1 = H - 1;
    if (box) {
        double R = sqrt(R2);
        double lo_x = floor((xp - R - ox) / cs) - 2.0, hi_x = ceil((xp + R - ox) / cs) + 2.0;
        double lo_y = floor((yp - R - oy) / cs) - 2.0, hi_y = ceil((yp + R - oy) / cs) + 2.0;
        if (hi_x < 0.0 || hi_y < 0.0 || lo_x > (double)(W - 1) || lo_y > (double)(H - 1)) return;
        if (lo_x > i0) i0 = (int32_t)lo_x;
        if (hi_x < i1) i1 = (int32_t)hi_x;
        if (lo_y > k0) k0 = (int32_t)lo_y;
        if (hi_y < k1) k1 = (int32_t)hi_y;
    }
    for (int32_t k = k0; k <= k1; ++k)
        for (int32_t i = i0; i <= i1; ++i) {
            double cx = ox + ((double)i + 0.5) * cs;
            double cy = oy + ((double)k + 0.5) * cs;
            double dx = cx - xp;
            double dy = cy - yp;
            if (dx * dx + dy * dy <= R2) stamp[(size_t)k * W + i] = 1;
        }
}

/* Stamp a single disk with the all-cells loop (pin P4 only). */
void orc_stamp_bruteforce(int32_t W, int32_t H, double cs, double ox, double oy,
                          double xp, double yp, double R2, uint8_t* stamp)
{
    orc_stamp_one(W, H, cs, ox, oy, xp, yp, R2, stamp, 0);
}

void orc_stamp_box(int32_t W, int32_t H, double cs, double ox, double oy,
                   double xp, double yp, double R2, uint8_t* stamp)
{
    orc_stamp_one(W, H, cs, ox, oy, xp, yp, R2, stamp, 1);
}

/* horizon_mode 0: Eq. 16 (C18); 1: time to reach the ring (orc_horizon_ring, f4).
 * footprint_mode 0: the j-step predicted covariance (C19); 1: the track's posterior covariance
 * P_k|k ("uncertainty given by Kalman filter at each step (Equation 12)", f4). */
int32_t orc_classify(int32_t W, int32_t H, double cs, double ox, double oy,
                     const uint8_t* static_mask, int32_t gx, int32_t gy,
                     double xr, double yr, double theta, double speed,
                     int32_t n, const double* tracks,
                     double dt, const double* Q, double w, double eps_v, double rs, int32_t hmax,
                     int32_t horizon_mode, int32_t footprint_mode,
                     uint8_t* cls, int32_t* t_out, int32_t* j_out, double* pred_out)
{
    if (W <= 0 || H <= 0 || cs <= 0.0 || n < 0) return ORC_E_INVALID_ARG;
    /* goal in bounds and not on a static wall */
    if (gx < 0 || gy < 0 || gx >= W || gy >= H) return ORC_E_OUT_OF_BOUNDS;
    if (static_mask[(size_t)gy * W + gx]) return ORC_E_OVERLAPPING;
    /* robot cell = floor((x_r - o_x) / cs) (S:41 floor binning) */
    double fxr = floor((xr - ox) / cs), fyr = floor((yr - oy) / cs);
    if (fxr < 0.0 || fyr < 0.0 || fxr >= (double)W || fyr >= (double)H) return ORC_E_OUT_OF_BOUNDS;
    int32_t rcx = (int32_t)fxr, rcy = (int32_t)fyr;
    if (static_mask[(size_t)rcy * W + rcx]) return ORC_E_INVALID_START;

    size_t ncell = (size_t)W * H;
    uint8_t* stamp = (uint8_t*)calloc(ncell, 1);
    if (!stamp) return ORC_E_INVALID_ARG;
    double c = cos(theta), s = sin(theta);
    for (int32_t i = 0; i < n; ++i) {
        const double* x = tracks + (size_t)i * 20;
        const double* P = x + 4;
        double rx = orc_warp_radius(xr, yr, c, s, x[0], x[1]);      /* O1, C24: from x_hat */
        int32_t t = orc_warp_number(rx, w);
        int32_t j = horizon_mode == 1 ? orc_horizon_ring(t, w, speed, dt, hmax)
                                       : orc_horizon(t, speed, x[2], x[3], eps_v, hmax);  /* O2 */
        double xo[4], Po[16];
        orc_predict(x, P, Q, dt, j, xo, Po);
        double R2 = orc_footprint_r2(footprint_mode == 1 ? P : Po, rs);
        if (t_out) t_out[i] = t;
        if (j_out) j_out[i] = j;
        if (pred_out) { pred_out[3 * i] = xo[0]; pred_out[3 * i + 1] = xo[1]; pred_out[3 * i + 2] = R2; }
        orc_stamp_one(W, H, cs, ox, oy, xo[0], xo[1], R2, stamp, 1);
    }
    int32_t status = ORC_OK;
    if (stamp[(size_t)gy * W + gx]) status = ORC_W_GOAL_SWALLOWED;
    /* precedence (C22): goal > robot-cell exemption > (static U stamped) > free */
    for (size_t q = 0; q < ncell; ++q)
        cls[q] = (static_mask[q] || stamp[q]) ? ORC_OBSTACLE : ORC_FREE;
    cls[(size_t)rcy * W + rcx] = ORC_FREE;
    cls[(size_t)gy * W + gx] = ORC_GOAL;
    free(stamp);
    return status;
}

/* Field initialisation in u-space (C7).
 * cold (u_prev == NULL): goal 1, obstacle 0, free 0.5 ("initialized with 0.5").
 * warm: fixed-now cells take their fixed value; every free cell keeps the value
 * it held after the previous tick ("the values evolve slowly
 * anyways"), so an obstacle cell released keeps u = 0 (phi = 1); the one
 * exception is a released goal (cls_prev GOAL, free now), which restarts at
 * u = 0 like a released obstacle instead of keeping u = 1: a free cell at the
 * maximum value would be a spurious maximum of the field, the very trap of the
 * descent walk that C7 avoids.  cls_prev may be NULL (no goal released). */
void orc_init_u32(int64_t ncell, const uint8_t* cls, const float* u_prev, const uint8_t* cls_prev, float* u)
{
    for (int64_t q = 0; q < ncell; ++q) {
        if (cls[q] == ORC_GOAL) u[q] = 1.0f;
        else if (cls[q] == ORC_OBSTACLE) u[q] = 0.0f;
        else if (u_prev == NULL) u[q] = 0.5f;
        else if (cls_prev != NULL && cls_prev[q] == ORC_GOAL) u[q] = 0.0f;
        else u[q] = u_prev[q];
    }
}

void orc_init_u64(int64_t ncell, const uint8_t* cls, double* u)
{
    for (int64_t q = 0; q < ncell; ++q)
        u[q] = cls[q] == ORC_GOAL ? 1.0 : (cls[q] == ORC_OBSTACLE ? 0.0 : 0.5);
}

/* ------------------------------------------------------------------------ */
/* O4-O5  red-black Gauss-Seidel relaxation + stop rule                     */
/* (Eqs. 1-2, Alg. 1; C1, C2, C4-C6)  */
/* ------------------------------------------------------------------------ */

/* Cells with cls != ORC_FREE are fixed (Dirichlet) and keep the value they
 * hold in u, so tests may pass general fixed values (pin P8).  Outside the
 * grid u = 0 (C4: outside = obstacle).  One sweep = red pass ((x+y) even, in
 * the grid's own coordinates) then black pass; each free cell becomes
 * 0.25 * ((E + W) + (N + S)) (C2).  res_s = max |new - old| over the free
 * cells of sweep s.  Stop after sweep s when (s % check_every == 0 and
 * res_s < tol) or s == max_sweeps.  Returns sweeps done; *res_out = res_s of
 * the last sweep (0 if none). */
/* General form used for row slabs: colour = parity of (x + row_parity + y); the residual is the
 * max over the free cells of rows [res_r0, res_r1) only (the owned rows of a slab). */
int32_t orc_relax_f32_ex(int32_t W, int32_t H, const uint8_t* cls, float* u, int32_t max_sweeps,
                         int32_t check_every, float tol, int32_t row_parity, int32_t res_r0, int32_t res_r1,
                         float* res_out)
{
    float res = 0.0f;
    int32_t s = 0;
    if (check_every < 1) check_every = 1;
    for (s = 1; s <= max_sweeps; ++s) {
        res = 0.0f;
        for (int color = 0; color < 2; ++color)
            for (int32_t y = 0; y < H; ++y)
                for (int32_t x = 0; x < W; ++x) {
                    if (((x + y + row_parity) & 1) != color) continue;
                    size_t q = (size_t)y * W + x;
                    if (cls[q] != ORC_FREE) continue;
                    float uE = x + 1 < W ? u[q + 1] : 0.0f;
                    float uW = x > 0 ? u[q - 1] : 0.0f;
                    float uN = y > 0 ? u[q - W] : 0.0f;
                    float uS = y + 1 < H ? u[q + W] : 0.0f;
                    float nv = 0.25f * ((uE + uW) + (uN + uS));
                    float d = fabsf(nv - u[q]);
                    if (d > res && y >= res_r0 && y < res_r1) res = d;
                    u[q] = nv;
                }
        if ((s % check_every == 0 && res < tol) || s == max_sweeps) break;
    }
    if (max_sweeps <= 0) { s = 0; res = 0.0f; }
    if (res_out) *res_out = res;
    return s;
}

int32_t orc_relax_f32(int32_t W, int32_t H, const uint8_t* cls, float* u,
                      int32_t max_sweeps, int32_t check_every, float tol, float* res_out)
{
    return orc_relax_f32_ex(W, H, cls, u, max_sweeps, check_every, tol, 0, 0, H, res_out);
}

/* orc_relax_f32 with each colour pass split over `threads` OpenMP threads by rows (timing variant,
 * SURVEY 8(c)).  The cells of one colour never neighbour each other, so within a pass every update
 * reads only the other colour and the pass is order-free; the residual is a max, which is exact in
 * any order.  Hence the result is bit-identical to the single-thread loop (pin P14). */
int32_t orc_relax_f32_omp(int32_t W, int32_t H, const uint8_t* cls, float* u, int32_t max_sweeps,
                          int32_t check_every, float tol, int32_t threads, float* res_out)
{
    float res = 0.0f;
    int32_t s = 0;
    if (check_every < 1) check_every = 1;
    if (threads < 1) threads = 1;
    for (s = 1; s <= max_sweeps; ++s) {
        res = 0.0f;
        for (int color = 0; color < 2; ++color) {
#pragma omp parallel for num_threads(threads) schedule(static) reduction(max : res)
            for (int32_t y = 0; y < H; ++y)
                for (int32_t x = (color + y) & 1; x < W; x += 2) {
                    size_t q = (size_t)y * W + x;
                    if (cls[q] != ORC_FREE) continue;
                    float uE = x + 1 < W ? u[q + 1] : 0.0f;
                    float uW = x > 0 ? u[q - 1] : 0.0f;
                    float uN = y > 0 ? u[q - W] : 0.0f;
                    float uS = y + 1 < H ? u[q + W] : 0.0f;
                    float nv = 0.25f * ((uE + uW) + (uN + uS));
                    float d = fabsf(nv - u[q]);
                    if (d > res) res = d;
                    u[q] = nv;
                }
        }
        if ((s % check_every == 0 && res < tol) || s == max_sweeps) break;
    }
    if (max_sweeps <= 0) { s = 0; res = 0.0f; }
    if (res_out) *res_out = res;
    return s;
}

int32_t orc_relax_f64(int32_t W, int32_t H, const uint8_t* cls, double* u,
                      int32_t max_sweeps, int32_t check_every, double tol, double* res_out)
{
    double res = 0.0;
    int32_t s = 0;
    if (check_every < 1) check_every = 1;
    for (s = 1; s <= max_sweeps; ++s) {
        res = 0.0;
        for (int color = 0; color < 2; ++color)
            for (int32_t y = 0; y < H; ++y)
                for (int32_t x = 0; x < W; ++x) {
                    if (((x + y) & 1) != color) continue;
                    size_t q = (size_t)y * W + x;
                    if (cls[q] != ORC_FREE) continue;
                    double uE = x + 1 < W ? u[q + 1] : 0.0;
                    double uW = x > 0 ? u[q - 1] : 0.0;
                    double uN = y > 0 ? u[q - W] : 0.0;
                    double uS = y + 1 < H ? u[q + W] : 0.0;
                    double nv = 0.25 * ((uE + uW) + (uN + uS));
                    double d = fabs(nv - u[q]);
                    if (d > res) res = d;
                    u[q] = nv;
                }
        if ((s % check_every == 0 && res < tol) || s == max_sweeps) break;
    }
    if (max_sweeps <= 0) { s = 0; res = 0.0; }
    if (res_out) *res_out = res;
    return s;
}

/* Jacobi, Eq. 1 literally: every free cell from the previous
 * iterate.  Oracle-only variant for pins P7 and P12 (Jacobi and red-black
 * share the fixed point). */
int32_t orc_jacobi_f64(int32_t W, int32_t H, const uint8_t* cls, double* u,
                       int32_t max_sweeps, double tol, double* res_out)
{
    size_t ncell = (size_t)W * H;
    double* old = (double*)malloc(ncell * sizeof(double));
    double res = 0.0;
    int32_t s = 0;
    for (s = 1; s <= max_sweeps; ++s) {
        memcpy(old, u, ncell * sizeof(double));
        res = 0.0;
        for (int32_t y = 0; y < H; ++y)
            for (int32_t x = 0; x < W; ++x) {
                size_t q = (size_t)y * W + x;
                if (cls[q] != ORC_FREE) continue;
                double uE = x + 1 < W ? old[q + 1] : 0.0;
                double uW = x > 0 ? old[q - 1] : 0.0;
                double uN = y > 0 ? old[q - W] : 0.0;
                double uS = y + 1 < H ? old[q + W] : 0.0;
                double nv = 0.25 * ((uE + uW) + (uN + uS));
                double d = fabs(nv - old[q]);
                if (d > res) res = d;
                u[q] = nv;
            }
        if (res < tol || s == max_sweeps) break;
    }
    if (max_sweeps <= 0) { s = 0; res = 0.0; }
    free(old);
    if (res_out) *res_out = res;
    return s;
}

/* Lexicographic Gauss-Seidel, Eq. 2 literally, in fp32: rows
 * y = 0..H-1, columns x = 0..W-1, in place, so W (x - 1) and N (y - 1) are this sweep's values and
 * E, S the previous sweep's; 0.25 * ((E + W) + (N + S)); residual and stop rule as orc_relax_f32. */
int32_t orc_relax_lex_f32(int32_t W, int32_t H, const uint8_t* cls, float* u, int32_t max_sweeps,
                          int32_t check_every, float tol, float* res_out)
{
    float res = 0.0f;
    int32_t s = 0;
    if (check_every < 1) check_every = 1;
    for (s = 1; s <= max_sweeps; ++s) {
        res = 0.0f;
        for (int32_t y = 0; y < H; ++y)
            for (int32_t x = 0; x < W; ++x) {
                size_t q = (size_t)y * W + x;
                if (cls[q] != ORC_FREE) continue;
                float uE = x + 1 < W ? u[q + 1] : 0.0f;
                float uW = x > 0 ? u[q - 1] : 0.0f;
                float uN = y > 0 ? u[q - W] : 0.0f;
                float uS = y + 1 < H ? u[q + W] : 0.0f;
                float nv = 0.25f * ((uE + uW) + (uN + uS));
                float d = fabsf(nv - u[q]);
                if (d > res) res = d;
                u[q] = nv;
            }
        if ((s % check_every == 0 && res < tol) || s == max_sweeps) break;
    }
    if (max_sweeps <= 0) { s = 0; res = 0.0f; }
    if (res_out) *res_out = res;
    return s;
}

/* Jacobi, Eq. 1 literally, in fp32: every free cell from the previous
 * iterate, 0.25 * ((E + W) + (N + S)); residual and stop rule as orc_relax_f32. */
int32_t orc_relax_jacobi_f32(int32_t W, int32_t H, const uint8_t* cls, float* u, int32_t max_sweeps,
                             int32_t check_every, float tol, float* res_out)
{
    size_t ncell = (size_t)W * H;
    float* old = (float*)malloc(ncell * sizeof(float));
    float res = 0.0f;
    int32_t s = 0;
    if (check_every < 1) check_every = 1;
    for (s = 1; s <= max_sweeps; ++s) {
        memcpy(old, u, ncell * sizeof(float));
        res = 0.0f;
        for (int32_t y = 0; y < H; ++y)
            for (int32_t x = 0; x < W; ++x) {
                size_t q = (size_t)y * W + x;
                if (cls[q] != ORC_FREE) continue;
                float uE = x + 1 < W ? old[q + 1] : 0.0f;
                float uW = x > 0 ? old[q - 1] : 0.0f;
                float uN = y > 0 ? old[q - W] : 0.0f;
                float uS = y + 1 < H ? old[q + W] : 0.0f;
                float nv = 0.25f * ((uE + uW) + (uN + uS));
                float d = fabsf(nv - old[q]);
                if (d > res) res = d;
                u[q] = nv;
            }
        if ((s % check_every == 0 && res < tol) || s == max_sweeps) break;
    }
    if (max_sweeps <= 0) { s = 0; res = 0.0f; }
    free(old);
    if (res_out) *res_out = res;
    return s;
}

/* Full-grid index matrix M_idx (Eq. 3; Alg. 1): per cell
 * 0..3 = the in-grid neighbour with the largest u in the order +x, -x, +y, -y (strict >), or
 * 4 goal, 5 obstacle, 6 no in-grid neighbour. */
void orc_index_matrix(int32_t W, int32_t H, const uint8_t* cls, const float* u, uint8_t* out)
{
    static const int dxs[4] = { +1, -1, 0, 0 };
    static const int dys[4] = { 0, 0, +1, -1 };
    for (int32_t y = 0; y < H; ++y)
        for (int32_t x = 0; x < W; ++x) {
            size_t q = (size_t)y * W + x;
            if (cls[q] == ORC_GOAL) { out[q] = 4; continue; }
            if (cls[q] == ORC_OBSTACLE) { out[q] = 5; continue; }
            int best_d = 6;
            float best = 0.0f;
            for (int d = 0; d < 4; ++d) {
                int nx = x + dxs[d], ny = y + dys[d];
                if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
                float v = u[(size_t)ny * W + nx];
                if (best_d == 6 || v > best) { best = v; best_d = d; }
            }
            out[q] = (uint8_t)best_d;
        }
}

/* Per-cell rubber band on the index matrix (Alg. 1 P:701-704 "for each cell in the index matrix in
 * parallel: calculate tension force T and potential force F via Eq. 6; update the index matrix with
 * the position of the neighbor with the minimum resultant force (Eqs. 4-5)"; reading
 * C37 of DESIGN.md).  A cell has one successor but possibly several predecessors, so the band acts on
 * the successor: for a free cell c with current successor m = M(c), each candidate n among its
 * in-grid, non-obstacle 4-neighbours is scored by the resultant force on n were the link c -> n ->
 * M(n):
 *   R(n) = F_vec + k_t (c - n) + k_t (M(n) - n),  F = 1/u(n) - 1/u(c),  F_vec = -F d (d = n - c,
 *   a unit axis vector; Eq. 6 in u-space as C13), where M(n) is the cell n's successor (n itself
 *   when n is the goal, an obstacle or has none: no tension from it);
 * candidates with u(n) <= 1e-9 or u(c) <= 1e-9 are skipped (C13).  The current successor is scored
 * first and kept on ties; the others follow in the order +x, -x, +y, -y with strict < (C8).  One
 * iteration updates the cells with (x + y) even, then those with (x + y) odd: a cell reads only its
 * neighbours' successors, which have the other colour, so each phase is order-free.  dir: H x W in/out,
 * codes of orc_index_matrix (0..3 = +x, -x, +y, -y; 4 goal, 5 obstacle, 6 none); goal, obstacle
 * and successor-less cells are not changed.  Parity pinned by hand (P27). */
void orc_cellband(int32_t W, int32_t H, const uint8_t* cls, const float* u, uint8_t* dir, int32_t iters, float kt)
{
    static const int dxs[4] = { +1, -1, 0, 0 };
    static const int dys[4] = { 0, 0, +1, -1 };
    for (int32_t it = 0; it < iters; ++it)
        for (int color = 0; color < 2; ++color)
            for (int32_t y = 0; y < H; ++y)
                for (int32_t x = 0; x < W; ++x) {
                    if (((x + y) & 1) != color) continue;
                    size_t q = (size_t)y * W + x;
                    if (cls[q] != ORC_FREE || dir[q] > 3) continue;
                    float uc = u[q];
                    if (uc <= 1e-9f) continue;
                    int best_d = dir[q];
                    float best = 0.0f;
                    int have = 0;
                    for (int pass = 0; pass < 5; ++pass) {
                        int d = pass == 0 ? dir[q] : pass - 1;
                        if (pass > 0 && d == dir[q]) continue;
                        int nx = x + dxs[d], ny = y + dys[d];
                        if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
                        size_t qn = (size_t)ny * W + nx;
                        if (cls[qn] == ORC_OBSTACLE) continue;
                        float un = u[qn];
                        if (un <= 1e-9f) continue;
                        int mx = nx, my = ny;  /* n's successor */
                        if (dir[qn] <= 3) { mx = nx + dxs[dir[qn]]; my = ny + dys[dir[qn]]; }
                        float F = 1.0f / un - 1.0f / uc;
                        float Rx = (-(F * (float)dxs[d]) + kt * (float)(x - nx)) + kt * (float)(mx - nx);
                        float Ry = (-(F * (float)dys[d]) + kt * (float)(y - ny)) + kt * (float)(my - ny);
                        float r2 = Rx * Rx + Ry * Ry;
                        if (!have || r2 < best) { best = r2; best_d = d; have = 1; }
                    }
                    dir[q] = (uint8_t)best_d;
                }
}

/* Walk along an index matrix (codes of orc_index_matrix) from (sx, sy): the cells visited, the start
 * included, until the goal (ORC_OK); an obstacle, a successor-less cell or more than max_len cells
 * is ORC_E_NO_PATH (*n_cells = 0).  Used to generate the path from the per-cell band's matrix
 * (Alg. 1 P:705 "Generate the current path based on the optimized index matrix"). */
int32_t orc_walk_dir(int32_t W, int32_t H, const uint8_t* dir, int32_t sx, int32_t sy, int32_t max_len,
                     int32_t* cells_xy, int32_t* n_cells)
{
    static const int dxs[4] = { +1, -1, 0, 0 };
    static const int dys[4] = { 0, 0, +1, -1 };
    int32_t n = 0, x = sx, y = sy;
    *n_cells = 0;
    if (max_len < 1) return ORC_E_NO_PATH;
    cells_xy[0] = x; cells_xy[1] = y; n = 1;
    for (;;) {
        uint8_t d = dir[(size_t)y * W + x];
        if (d == 4) { *n_cells = n; return ORC_OK; }
        if (d > 3) return ORC_E_NO_PATH;
        if (n + 1 > max_len) return ORC_E_NO_PATH;
        x += dxs[d]; y += dys[d];
        cells_xy[2 * n] = x; cells_xy[2 * n + 1] = y; ++n;
    }
}

/* Per-cell warp number (the paper's kernel 1, "calculate the warp of each cell"; the
 * numbered ellipses of Fig. warps): t of an obstacle at the cell centre. */
void orc_warp_map(int32_t W, int32_t H, double cs, double ox, double oy, double xr, double yr, double theta,
                  double w, int32_t* out)
{
    double c = cos(theta), s = sin(theta);
    for (int32_t y = 0; y < H; ++y)
        for (int32_t x = 0; x < W; ++x) {
            double px = ox + ((double)x + 0.5) * cs, py = oy + ((double)y + 0.5) * cs;
            out[(size_t)y * W + x] = orc_warp_number(orc_warp_radius(xr, yr, c, s, px, py), w);
        }
}

/* ------------------------------------------------------------------------ */
/* O6  descent walk on the implicit index matrix                            */
/* (Eq. 3, Alg. 1; C8, C9)   */
/* ------------------------------------------------------------------------ */

/* Eq. 3's argmin of phi is the argmax of u = 1 - phi.  From the robot cell:
 *   if c is the goal: done; if c is an obstacle: NoPath;
 *   n = in-bounds 4-neighbour with the largest u, scanned [+x, -x, +y, -y],
 *       replaced only on strictly greater (first maximum wins);
 *   append n; if the path is longer than max_len: NoPath.
 * On NoPath *n_cells = 0.  cells_xy holds max_len (x, y) pairs. */
int32_t orc_walk(int32_t W, int32_t H, const uint8_t* cls, const float* u,
                 int32_t sx, int32_t sy, int32_t max_len, int32_t* cells_xy, int32_t* n_cells)
{
    static const int dxs[4] = { +1, -1, 0, 0 };
    static const int dys[4] = { 0, 0, +1, -1 };
    int32_t n = 0, x = sx, y = sy;
    *n_cells = 0;
    if (max_len < 1) return ORC_E_NO_PATH;
    cells_xy[0] = x; cells_xy[1] = y; n = 1;
    for (;;) {
        uint8_t k = cls[(size_t)y * W + x];
        if (k == ORC_GOAL) { *n_cells = n; return ORC_OK; }
        if (k == ORC_OBSTACLE) return ORC_E_NO_PATH;
        int bx = -1, by = -1;
        float best = 0.0f;
        int have = 0;
        for (int d = 0; d < 4; ++d) {
            int nx = x + dxs[d], ny = y + dys[d];
            if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
            float v = u[(size_t)ny * W + nx];
            if (!have || v > best) { best = v; bx = nx; by = ny; have = 1; }
        }
        if (!have) return ORC_E_NO_PATH; /* 1x1 grid with a free cell */
        if (n + 1 > max_len) return ORC_E_NO_PATH;
        x = bx; y = by;
        cells_xy[2 * n] = x; cells_xy[2 * n + 1] = y; ++n;
    }
}

/* ------------------------------------------------------------------------ */
/* O7  rubber band (Eqs. 4-6, Fig. 1)        */
/* ------------------------------------------------------------------------ */

/* u at a continuous position (cell units) by bilinear interpolation of the
 * cell-centred samples at (i + 0.5, k + 0.5); samples outside the grid are 0
 * (C4, C14).  Evaluated as (1-ty)((1-tx)u00 + tx u10) + ty((1-tx)u01 + tx u11). */
static float orc_u_at(int32_t W, int32_t H, const float* u, int32_t i, int32_t k)
{
    if (i < 0 || k < 0 || i >= W || k >= H) return 0.0f;
    return u[(size_t)k * W + i];
}

float orc_bilerp(int32_t W, int32_t H, const float* u, float px, float py)
{
    float fx = px - 0.5f, fy = py - 0.5f;
    float x0f = floorf(fx), y0f = floorf(fy);
    float tx = fx - x0f, ty = fy - y0f;
    int32_t x0 = (int32_t)x0f, y0 = (int32_t)y0f;
    float u00 = orc_u_at(W, H, u, x0, y0);
    float u10 = orc_u_at(W, H, u, x0 + 1, y0);
    float u01 = orc_u_at(W, H, u, x0, y0 + 1);
    float u11 = orc_u_at(W, H, u, x0 + 1, y0 + 1);
    float a = (1.0f - tx) * u00 + tx * u10;
    float b = (1.0f - tx) * u01 + tx * u11;
    return (1.0f - ty) * a + ty * b;
}

/* One waypoint update (Eq. 4 argmin over the current position and 8 offsets
 * of length `step` (C12); Eq. 5 moves the waypoint there).
 * Tensions T = k_t (w_{i+-1} - c) (C11).  Eq. 6 in u-space:
 * F = 1/u(c) - 1/u(w_i) (P:311-313 with 1 - phi = u), acting along the
 * candidate direction d_hat with F_vec = -F d_hat (C13); candidates whose
 * cell is off-grid or an obstacle, or with u <= 1e-9, are skipped (S:208,
 * S:216-217).  The current position (F_vec = 0) wins all ties. */
static void orc_band_point(int32_t W, int32_t H, const uint8_t* cls, const float* u,
                           const float* wp, const float* wi, const float* wn,
                           float step, float kt, float* out)
{
    static const float ox[8] = { +1.f, -1.f, 0.f, 0.f, +1.f, +1.f, -1.f, -1.f };
    static const float oy[8] = { 0.f, 0.f, +1.f, -1.f, +1.f, -1.f, +1.f, -1.f };
    float bx = wi[0], by = wi[1];
    float tx = kt * (wp[0] - wi[0]) + kt * (wn[0] - wi[0]);
    float ty = kt * (wp[1] - wi[1]) + kt * (wn[1] - wi[1]);
    float best = tx * tx + ty * ty;
    float uw = orc_bilerp(W, H, u, wi[0], wi[1]);
    for (int d = 0; d < 8; ++d) {
        float cx = wi[0] + step * ox[d];
        float cy = wi[1] + step * oy[d];
        float fcx = floorf(cx), fcy = floorf(cy);
        if (fcx < 0.0f || fcy < 0.0f || fcx >= (float)W || fcy >= (float)H) continue;
        if (cls[(size_t)(int32_t)fcy * W + (int32_t)fcx] == ORC_OBSTACLE) continue;
        float uc = orc_bilerp(W, H, u, cx, cy);
        if (uc <= 1e-9f || uw <= 1e-9f) continue;
        float F = 1.0f / uc - 1.0f / uw;
        float hx = d < 4 ? ox[d] : ox[d] * 0.70710678f;
        float hy = d < 4 ? oy[d] : oy[d] * 0.70710678f;
        float Rx = (-(F * hx) + kt * (wp[0] - cx)) + kt * (wn[0] - cx);
        float Ry = (-(F * hy) + kt * (wp[1] - cy)) + kt * (wn[1] - cy);
        float r2 = Rx * Rx + Ry * Ry;
        if (r2 < best) { best = r2; bx = cx; by = cy; }
    }
    out[0] = bx; out[1] = by;
}

/* I iterations; each iteration updates the odd interior waypoints, then the
 * even ones (C10: parity order; the two waypoints each one reads are of the
 * other parity, so in-place update equals "reads before the phase").
 * Endpoints never move. w: n (x, y) pairs in cell units, in/out. */
void orc_band(int32_t W, int32_t H, const uint8_t* cls, const float* u,
              int32_t n, float* w, int32_t iters, float step, float kt)
{
    for (int32_t it = 0; it < iters; ++it)
        for (int p = 1; p >= 0; --p)
            for (int32_t i = 1; i + 1 < n; ++i) {
                if ((i & 1) != p) continue;
                float o[2];
                orc_band_point(W, H, cls, u, w + 2 * (i - 1), w + 2 * i, w + 2 * (i + 1), step, kt, o);
                w[2 * i] = o[0]; w[2 * i + 1] = o[1];
            }
}

/* orc_band with each parity phase split over `threads` OpenMP threads (timing variant): the
 * waypoints of one parity read only waypoints of the other parity, so a phase is order-free and
 * the result is bit-identical to orc_band (pin P14). */
void orc_band_omp(int32_t W, int32_t H, const uint8_t* cls, const float* u,
                  int32_t n, float* w, int32_t iters, float step, float kt, int32_t threads)
{
    if (threads < 1) threads = 1;
    for (int32_t it = 0; it < iters; ++it)
        for (int p = 1; p >= 0; --p) {
#pragma omp parallel for num_threads(threads) schedule(static)
            for (int32_t i = 1 + (p == 0); i < n - 1; i += 2) {
                float o[2];
                orc_band_point(W, H, cls, u, w + 2 * (i - 1), w + 2 * i, w + 2 * (i + 1), step, kt, o);
                w[2 * i] = o[0]; w[2 * i + 1] = o[1];
            }
        }
}

/* Resample (C15): each segment of length l is replaced by
 * ceil(max(l, 1)) equal sub-steps p = w_i + (k / m) (w_{i+1} - w_i); the
 * last waypoint is appended.  Returns the number of points (only the first
 * max_out are written). */
int32_t orc_resample(int32_t n, const float* w, int32_t max_out, float* out)
{
    int32_t cnt = 0;
    if (n <= 0) return 0;
    for (int32_t i = 0; i + 1 < n; ++i) {
        float dx = w[2 * (i + 1)] - w[2 * i];
        float dy = w[2 * (i + 1) + 1] - w[2 * i + 1];
        float l = sqrtf(dx * dx + dy * dy);
        int32_t m = (int32_t)ceilf(l > 1.0f ? l : 1.0f);
        for (int32_t k = 0; k < m; ++k) {
            float t = (float)k / (float)m;
            if (cnt < max_out) {
                out[2 * cnt] = w[2 * i] + t * dx;
                out[2 * cnt + 1] = w[2 * i + 1] + t * dy;
            }
            ++cnt;
        }
    }
    if (cnt < max_out) { out[2 * cnt] = w[2 * (n - 1)]; out[2 * cnt + 1] = w[2 * (n - 1) + 1]; }
    ++cnt;
    return cnt;
}

/* O8 (Alg. 1 P:705-706 "Move the robot to the next cell on the current path";
 * S:233): the first resampled waypoint at distance >= 1 cell from the first
 * one (the robot's cell centre), else the last (the goal). */
int32_t orc_next_waypoint(int32_t n, const float* pts, float* nx, float* ny)
{
    if (n <= 0) return -1;
    for (int32_t i = 1; i < n; ++i) {
        float dx = pts[2 * i] - pts[0];
        float dy = pts[2 * i + 1] - pts[1];
        if (dx * dx + dy * dy >= 1.0f) { *nx = pts[2 * i]; *ny = pts[2 * i + 1]; return i; }
    }
    *nx = pts[2 * (n - 1)]; *ny = pts[2 * (n - 1) + 1];
    return n - 1;
}

/* ------------------------------------------------------------------------ */
/* f1  Kalman update, association, spawn/prune (the step before a1)         */
/* (Eqs. 11-13; H of P:558-565; R = sigma_z^2 I, P:569-572 and    */
/* S:307; association and track management S:281-298, C28-C30)             */
/* ------------------------------------------------------------------------ */

enum { ORC_W_TRUNCATED = 2, ORC_W_SINGULAR = 3 };

/* Eqs. 11-13 written out with the explicit H = [I2 0]:
 *   K = P H^T (H P H^T + R)^-1;  x <- x + K (z - H x);  P <- (I - K H) P,
 * then P <- (P + P^T) / 2 (C28).  The 2x2 inverse is the adjugate over the
 * determinant.  Returns 0, or -1 (x, P untouched) when H P H^T + R is not
 * positive definite (S:276 SingularInnovation). */
int32_t orc_kalman_update(double* x, double* P, const double* z, const double* R)
{
    static const double Hm[8] = { 1.0, 0.0, 0.0, 0.0,
                                  0.0, 1.0, 0.0, 0.0 };
    double Hx[2], y[2], HP[8], S[4], Si[4], PHt[8], K[8], IKH[16], Pn[16], xn[4];
    for (int r = 0; r < 2; ++r) {
        double acc = 0.0;
        for (int k = 0; k < 4; ++k) acc = acc + Hm[r * 4 + k] * x[k];
        Hx[r] = acc;
        y[r] = z[r] - Hx[r];
    }
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 4; ++k) acc = acc + Hm[r * 4 + k] * P[k * 4 + c];
            HP[r * 4 + c] = acc;
        }
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 4; ++k) acc = acc + HP[r * 4 + k] * Hm[c * 4 + k];
            S[r * 2 + c] = acc + R[r * 2 + c];
        }
    double det = S[0] * S[3] - S[1] * S[2];
    if (!(det > 0.0) || !(S[0] > 0.0) || !(det < 1.0e300)) return -1;
    Si[0] = S[3] / det;
    Si[1] = -S[1] / det;
    Si[2] = -S[2] / det;
    Si[3] = S[0] / det;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 2; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 4; ++k) acc = acc + P[r * 4 + k] * Hm[c * 4 + k];
            PHt[r * 2 + c] = acc;
        }
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 2; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 2; ++k) acc = acc + PHt[r * 2 + k] * Si[k * 2 + c];
            K[r * 2 + c] = acc;
        }
    for (int r = 0; r < 4; ++r) {
        double acc = 0.0;
        for (int k = 0; k < 2; ++k) acc = acc + K[r * 2 + k] * y[k];
        xn[r] = x[r] + acc;
    }
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 2; ++k) acc = acc + K[r * 2 + k] * Hm[k * 4 + c];
            IKH[r * 4 + c] = (r == c ? 1.0 : 0.0) - acc;
        }
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 4; ++k) acc = acc + IKH[r * 4 + k] * P[k * 4 + c];
            Pn[r * 4 + c] = acc;
        }
    for (int r = 0; r < 4; ++r) x[r] = xn[r];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) P[r * 4 + c] = 0.5 * (Pn[r * 4 + c] + Pn[c * 4 + r]);
    return 0;
}

/* Greedy gated nearest neighbour (the paper is silent, C29):
 * repeatedly take the globally closest still-free (track, detection) pair
 * with squared distance dx*dx + dy*dy <= gate^2 (dx = z_x - x_pred), ties to
 * the lower track index, then the lower detection index.  pxy[2 n] predicted
 * positions, z[2 m] detections; match_t[n] = detection or -1; det_used[m]. */
void orc_associate(int32_t n, const double* pxy, int32_t m, const double* z, double gate,
                   int32_t* match_t, uint8_t* det_used)
{
    double g2 = gate * gate;
    for (int32_t i = 0; i < n; ++i) match_t[i] = -1;
    for (int32_t j = 0; j < m; ++j) det_used[j] = 0;
    for (;;) {
        int32_t bi = -1, bj = -1;
        double bd = 0.0;
        for (int32_t i = 0; i < n; ++i) {
            if (match_t[i] >= 0) continue;
            for (int32_t j = 0; j < m; ++j) {
                if (det_used[j]) continue;
                double dx = z[2 * j] - pxy[2 * i];
                double dy = z[2 * j + 1] - pxy[2 * i + 1];
                double d2 = dx * dx + dy * dy;
                if (d2 <= g2 && (bi < 0 || d2 < bd)) { bd = d2; bi = i; bj = j; }
            }
        }
        if (bi < 0) break;
        match_t[bi] = bj;
        det_used[bj] = 1;
    }
}

/* One tracker tick (Alg. 1 P:680-688 "Read ... Detect ... Estimate", C30):
 *   1. predict every track one step (Eqs. 9-10, orc_predict with j = 1);
 *   2. associate detections with the predicted positions (orc_associate);
 *   3. matched: Eqs. 11-13 with R = sigma_z^2 I, missed = 0 (singular
 *      innovation: keeps the prediction, missed + 1, warning);
 *      unmatched: keeps the prediction, missed + 1;
 *   4. prune tracks with missed > prune_after, keeping the order;
 *   5. append one track per unmatched detection in detection order:
 *      x = (z, 0, 0), P = diag(var_pos, var_pos, var_vel, var_vel);
 *   6. keep at most max_tracks (> 0) tracks, survivors first (warning).
 * trk[cap][20] (x[4], P[16]) and missed[cap] in/out, cap >= n + m.
 * Returns ORC_OK, ORC_W_TRUNCATED or ORC_W_SINGULAR (the larger code wins). */
int32_t orc_track_step(int32_t n, double* trk, int32_t* missed, int32_t cap, int32_t m, const double* z,
                       double dt, const double* Q, double sigma_z, double gate, double var_pos,
                       double var_vel, int32_t prune_after, int32_t max_tracks, int32_t* n_out)
{
    int32_t status = ORC_OK;
    double* pred = (double*)malloc(sizeof(double) * 20 * (size_t)(n > 0 ? n : 1));
    double* pxy = (double*)calloc(2 * (size_t)(n > 0 ? n : 1), sizeof(double));
    int32_t* mt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t* mis = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    uint8_t* du = (uint8_t*)malloc((size_t)(m > 0 ? m : 1));
    double R[4] = { sigma_z * sigma_z, 0.0, 0.0, sigma_z * sigma_z };
    for (int32_t i = 0; i < n; ++i) {
        orc_predict(trk + 20 * i, trk + 20 * i + 4, Q, dt, 1, pred + 20 * i, pred + 20 * i + 4);
        pxy[2 * i] = pred[20 * i];
        pxy[2 * i + 1] = pred[20 * i + 1];
    }
    orc_associate(n, pxy, m, z, gate, mt, du);
    for (int32_t i = 0; i < n; ++i) {
        mis[i] = missed[i] + 1;
        if (mt[i] >= 0) {
            if (orc_kalman_update(pred + 20 * i, pred + 20 * i + 4, z + 2 * mt[i], R) == 0) mis[i] = 0;
            else status = ORC_W_SINGULAR;
        }
    }
    int32_t limit = max_tracks > 0 ? max_tracks : cap;
    if (limit > cap) limit = cap;
    int32_t k = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (mis[i] > prune_after) continue;
        if (k >= limit) { if (status < ORC_W_TRUNCATED) status = ORC_W_TRUNCATED; continue; }
        memcpy(trk + 20 * k, pred + 20 * i, 20 * sizeof(double));
        missed[k] = mis[i];
        ++k;
    }
    for (int32_t j = 0; j < m; ++j) {
        if (du[j]) continue;
        if (k >= limit) { if (status < ORC_W_TRUNCATED) status = ORC_W_TRUNCATED; continue; }
        double* t = trk + 20 * k;
        memset(t, 0, 20 * sizeof(double));
        t[0] = z[2 * j];
        t[1] = z[2 * j + 1];
        t[4 + 0] = var_pos;
        t[4 + 5] = var_pos;
        t[4 + 10] = var_vel;
        t[4 + 15] = var_vel;
        missed[k] = 0;
        ++k;
    }
    *n_out = k;
    free(pred); free(pxy); free(mt); free(mis); free(du);
    return status;
}

/* ------------------------------------------------------------------------ */
/* f2  closed-loop simulator ("Move the robot",       */
/* P:758-768 the success protocol, P:538-540 obstacle motion;    */
/* readings C31-C35).  Only + - * / sqrt floor, so the CUDA simulator can   */
/* be bit-identical; randomness is the counter-based generator below, which */
/* the CUDA side implements independently.                                  */
/* ------------------------------------------------------------------------ */

static uint64_t orc_splitmix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Uniform in [0, 1) with 53 random bits, a pure function of the counters (C31). */
double orc_rng_u01(uint64_t seed, uint64_t trial, uint64_t tick, uint64_t entity, uint64_t k)
{
    uint64_t h = orc_splitmix(seed ^ orc_splitmix(trial ^ orc_splitmix(tick ^ orc_splitmix(entity * 64u + k))));
    return (double)(h >> 11) * 0x1.0p-53;
}

/* Approximately standard normal: Irwin-Hall sum of 12 uniforms minus 6 (C31). */
double orc_rng_normal(uint64_t seed, uint64_t trial, uint64_t tick, uint64_t entity, uint64_t stream)
{
    double s = 0.0;
    for (uint64_t i = 0; i < 12; ++i) s = s + orc_rng_u01(seed, trial, tick, entity, stream * 16u + i);
    return s - 6.0;
}

/* Detections of tick `tick` (C32): every obstacle, in index order, at its true position plus
 * sigma_z N(0,1) per axis (streams 1, 2). z[2 n]. */
void orc_sim_sense(int32_t n, const double* obs, double sigma_z, uint64_t seed, uint64_t trial, uint64_t tick,
                   double* z)
{
    for (int32_t i = 0; i < n; ++i) {
        z[2 * i] = obs[4 * i] + sigma_z * orc_rng_normal(seed, trial, tick, (uint64_t)i, 1);
        z[2 * i + 1] = obs[4 * i + 1] + sigma_z * orc_rng_normal(seed, trial, tick, (uint64_t)i, 2);
    }
}

static int orc_blocked(int32_t W, int32_t H, double cs, double ox, double oy, const uint8_t* mask, double px,
                       double py)
{
    double fx = floor((px - ox) / cs), fy = floor((py - oy) / cs);
    if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)W && fy < (double)H)) return 1;
    return mask[(size_t)fy * W + (size_t)fx] != 0;
}

/* Any sample p + (k / m) td u, k = 1..m, m = ceil(td / (cs / 2)), blocked (C34: thin walls are
 * not jumped over). */
static int orc_probe(int32_t W, int32_t H, double cs, double ox, double oy, const uint8_t* mask, double x,
                     double y, double ux, double uy, double td)
{
    int32_t m = (int32_t)ceil(td / (0.5 * cs));
    for (int32_t k = 1; k <= m; ++k) {
        double d = td * (double)k / (double)m;
        if (orc_blocked(W, H, cs, ox, oy, mask, x + ux * d, y + uy * d)) return 1;
    }
    return 0;
}

/* One simulator tick for one trial (C33-C35), after the planner produced waypoint (wp_x, wp_y)
 * in cell units (has_wp = 0: the walk failed -- the robot keeps its heading):
 *   robot: heading turns toward the waypoint by at most the angle whose cosine/sine are
 *     cfg[6], cfg[7], renormalised; position advances speed dt (never stops);
 *     turning-angle histogram bin k: the largest k with dot(h_old, h_new) <= cos_bins[k];
 *   obstacles (Jacobi: every rule reads the tick-start positions): heading jitter by the
 *     rational (Cayley) rotation with a = sigma_h N / 2 (stream 0); turn away from the first
 *     other obstacle within 2 r_o + turn_dist that lies ahead (reflection about the centre
 *     line); turn away from walls probed up to turn_dist ahead per axis (orc_probe;
 *     reflection), speed restored,
 *     move v dt, clamp into [r_o, extent - r_o];
 *   status: collision (robot centre outside the grid, a wall cell centre within r_r, or an
 *     obstacle centre closer than r_r + r_o) before success (within goal_r of the goal); then
 *     timeout at max_ticks (P:758-763 strict criterion).
 * rob[6] = x, y, hx, hy, speed, length; obs[n][4] = x, y, vx, vy; obs_speed[n];
 * cfg = dt, r_robot, r_obs, goal_r, turn_dist, sigma_h, cos_d, sin_d. */
void orc_sim_move(int32_t W, int32_t H, double cs, double ox, double oy, const uint8_t* mask, double* rob,
                  int32_t* ticks, int32_t* status, double goal_x, double goal_y, int32_t has_wp, double wp_x,
                  double wp_y, int32_t n, double* obs, const double* obs_speed, const double* cfg,
                  int32_t max_ticks, uint64_t seed, uint64_t trial, const double* cos_bins, int32_t* hist)
{
    const double dt = cfg[0], rr = cfg[1], ro = cfg[2], gr = cfg[3], td = cfg[4], sh = cfg[5];
    const double cd = cfg[6], sd = cfg[7];
    const uint64_t tick = (uint64_t)*ticks;
    /* robot */
    double hx = rob[2], hy = rob[3];
    double nhx = hx, nhy = hy;
    if (has_wp) {
        double dx = (ox + wp_x * cs) - rob[0];
        double dy = (oy + wp_y * cs) - rob[1];
        double l2 = dx * dx + dy * dy;
        if (l2 > 0.0) {
            double l = sqrt(l2);
            double ux = dx / l, uy = dy / l;
            double dot = hx * ux + hy * uy;
            if (dot >= cd) {
                nhx = ux;
                nhy = uy;
            } else {
                double sg = (hx * uy - hy * ux) >= 0.0 ? 1.0 : -1.0;
                nhx = hx * cd - sg * (hy * sd);
                nhy = sg * (hx * sd) + hy * cd;
            }
            double nn = sqrt(nhx * nhx + nhy * nhy);
            nhx = nhx / nn;
            nhy = nhy / nn;
        }
    }
    double dturn = hx * nhx + hy * nhy;
    int32_t bin = 0;
    for (int32_t k = 35; k >= 0; --k)
        if (dturn <= cos_bins[k]) { bin = k; break; }
    hist[bin] += 1;
    const double step = rob[4] * dt;
    rob[0] = rob[0] + step * nhx;
    rob[1] = rob[1] + step * nhy;
    rob[2] = nhx;
    rob[3] = nhy;
    rob[5] = rob[5] + step;
    /* obstacles, from the tick-start positions */
    double* old = (double*)malloc(sizeof(double) * 4 * (size_t)(n > 0 ? n : 1));
    memcpy(old, obs, sizeof(double) * 4 * (size_t)n);
    const double xmax = ox + (double)W * cs, ymax = oy + (double)H * cs;
    for (int32_t i = 0; i < n; ++i) {
        double x = old[4 * i], y = old[4 * i + 1], vx = old[4 * i + 2], vy = old[4 * i + 3];
        double a = 0.5 * sh * orc_rng_normal(seed, trial, tick, (uint64_t)i, 0);
        double a2 = a * a;
        double c = (1.0 - a2) / (1.0 + a2), s = (2.0 * a) / (1.0 + a2);
        double rvx = c * vx - s * vy, rvy = s * vx + c * vy;
        vx = rvx;
        vy = rvy;
        const double lim = 2.0 * ro + td;
        for (int32_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = old[4 * j] - x, dy = old[4 * j + 1] - y;
            double d2 = dx * dx + dy * dy;
            if (d2 < lim * lim && d2 > 0.0 && dx * vx + dy * vy > 0.0) {
                double d = sqrt(d2);
                double nx = dx / d, ny = dy / d;
                double vn = vx * nx + vy * ny;
                vx = vx - 2.0 * vn * nx;
                vy = vy - 2.0 * vn * ny;
                break;
            }
        }
        double vs = sqrt(vx * vx + vy * vy);
        if (vs > 0.0) {
            double ux = vx / vs, uy = vy / vs;
            int bx = orc_probe(W, H, cs, ox, oy, mask, x, y, ux, 0.0, td);
            int by = orc_probe(W, H, cs, ox, oy, mask, x, y, 0.0, uy, td);
            if (bx) vx = -vx;
            if (by) vy = -vy;
            if (!bx && !by && orc_probe(W, H, cs, ox, oy, mask, x, y, ux, uy, td)) {
                vx = -vx;
                vy = -vy;
            }
            double f = obs_speed[i] / vs;
            vx = vx * f;
            vy = vy * f;
        }
        x = x + vx * dt;
        y = y + vy * dt;
        if (x < ox + ro) { x = ox + ro; vx = fabs(vx); }
        if (x > xmax - ro) { x = xmax - ro; vx = -fabs(vx); }
        if (y < oy + ro) { y = oy + ro; vy = fabs(vy); }
        if (y > ymax - ro) { y = ymax - ro; vy = -fabs(vy); }
        obs[4 * i] = x;
        obs[4 * i + 1] = y;
        obs[4 * i + 2] = vx;
        obs[4 * i + 3] = vy;
    }
    free(old);
    /* status */
    const double x = rob[0], y = rob[1];
    int coll = !(x >= ox && y >= oy && x < xmax && y < ymax);
    if (!coll) {
        int32_t cx0 = (int32_t)floor((x - rr - ox) / cs), cx1 = (int32_t)floor((x + rr - ox) / cs);
        int32_t cy0 = (int32_t)floor((y - rr - oy) / cs), cy1 = (int32_t)floor((y + rr - oy) / cs);
        for (int32_t cy = cy0; cy <= cy1 && !coll; ++cy)
            for (int32_t cx = cx0; cx <= cx1 && !coll; ++cx) {
                if (cx < 0 || cy < 0 || cx >= W || cy >= H) continue;
                if (!mask[(size_t)cy * W + cx]) continue;
                double ddx = (ox + ((double)cx + 0.5) * cs) - x, ddy = (oy + ((double)cy + 0.5) * cs) - y;
                if (ddx * ddx + ddy * ddy <= rr * rr) coll = 1;
            }
    }
    for (int32_t j = 0; j < n && !coll; ++j) {
        double dx = obs[4 * j] - x, dy = obs[4 * j + 1] - y;
        double lim = rr + ro;
        if (dx * dx + dy * dy < lim * lim) coll = 1;
    }
    *ticks = *ticks + 1;
    if (coll) *status = 2;
    else if ((x - goal_x) * (x - goal_x) + (y - goal_y) * (y - goal_y) <= gr * gr) *status = 1;
    else if (*ticks >= max_ticks) *status = 3;
}
