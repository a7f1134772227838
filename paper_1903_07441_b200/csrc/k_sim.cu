// Row f2: the closed-loop simulator around Algorithm 1 -- the step after a9
// ("Move the robot") and the world the paper's success protocol runs in.
// Batched: one thread per trial moves its robot and obstacles and checks the trial status; one
// thread per (trial, obstacle) produces the next tick's detections.
//
//   k_sim_move   robot turns toward the planner's next waypoint (at most turn_max per tick) and
//                advances speed dt; obstacles jitter (Cayley rotation), turn away from obstacles
//                ahead and from walls, move, clamp; collision / success / timeout (C33-C35)
//   k_sim_sense  detections = true positions + det_sigma N(0, 1) (C32)
//
// Randomness: the counter-based generator of C31 (splitmix64 chain, Irwin-Hall normal), written
// here independently of the oracle's.  Arithmetic: + - * / sqrt floor only, fp64, so the result is
// bit-identical to oracle/twg_oracle.c (orc_sim_move, orc_sim_sense) under -fmad=false.
#include "twg_kernels.cuh"

namespace twg {

__device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double rng_u01(uint64_t seed, uint64_t trial, uint64_t tick, uint64_t entity, uint64_t k) {
    const uint64_t h = sm64(seed ^ sm64(trial ^ sm64(tick ^ sm64(entity * 64u + k))));
    return (double)(h >> 11) * 0x1.0p-53;
}

__device__ double rng_normal(uint64_t seed, uint64_t trial, uint64_t tick, uint64_t entity, uint64_t stream) {
    double s = 0.0;
    for (uint64_t i = 0; i < 12; ++i) s = s + rng_u01(seed, trial, tick, entity, stream * 16u + i);
    return s - 6.0;
}

__device__ __forceinline__ bool sim_blocked(const SimArgs& a, const uint8_t* mask, double px, double py) {
    const double fx = floor((px - a.ox) / a.cs), fy = floor((py - a.oy) / a.cs);
    if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)a.W && fy < (double)a.H)) return true;
    return mask[(int64_t)fy * a.W + (int64_t)fx] != 0;
}

// Any sample p + (k / m) td u, k = 1..m, m = ceil(td / (cs / 2)), blocked (C34).
__device__ bool sim_probe(const SimArgs& a, const uint8_t* mask, double x, double y, double ux, double uy,
                          double td) {
    const int m = (int)ceil(td / (0.5 * a.cs));
    for (int k = 1; k <= m; ++k) {
        const double d = td * (double)k / (double)m;
        if (sim_blocked(a, mask, x + ux * d, y + uy * d)) return true;
    }
    return false;
}

__global__ void k_sim_move(SimArgs a) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= a.B || a.status[b] != 0) return;
    const uint8_t* mask = a.mask + (int64_t)b * a.H * a.W;
    double* rob = a.rob + (int64_t)b * 6;
    const int n = a.n_obs[b];
    double* obs = a.obs + (int64_t)b * a.ocap * 4;
    double* old = a.obs_old + (int64_t)b * a.ocap * 4;
    const uint64_t tick = (uint64_t)a.ticks[b];
    const uint64_t trial = (uint64_t)b;
    // robot: turn toward the next waypoint of this tick's plan (walk failed: keep the heading)
    const double hx = rob[2], hy = rob[3];
    double nhx = hx, nhy = hy;
    const PathMeta& pm = a.meta[b];
    if (pm.status == 0) {
        const double dx = (a.ox + (double)pm.next_x * a.cs) - rob[0];
        const double dy = (a.oy + (double)pm.next_y * a.cs) - rob[1];
        const double l2 = dx * dx + dy * dy;
        if (l2 > 0.0) {
            const double l = sqrt(l2);
            const double ux = dx / l, uy = dy / l;
            const double dot = hx * ux + hy * uy;
            if (dot >= a.cos_d) {
                nhx = ux;
                nhy = uy;
            } else {
                const double sg = (hx * uy - hy * ux) >= 0.0 ? 1.0 : -1.0;
                nhx = hx * a.cos_d - sg * (hy * a.sin_d);
                nhy = sg * (hx * a.sin_d) + hy * a.cos_d;
            }
            const double nn = sqrt(nhx * nhx + nhy * nhy);
            nhx = nhx / nn;
            nhy = nhy / nn;
        }
    }
    const double dturn = hx * nhx + hy * nhy;
    int bin = 0;
    for (int k = 35; k >= 0; --k)
        if (dturn <= a.cos_bins[k]) {
            bin = k;
            break;
        }
    a.hist[(int64_t)b * 36 + bin] += 1;
    const double step = rob[4] * a.dt;
    rob[0] = rob[0] + step * nhx;
    rob[1] = rob[1] + step * nhy;
    rob[2] = nhx;
    rob[3] = nhy;
    rob[5] = rob[5] + step;
    // obstacles, every rule reading the tick-start positions
    for (int q = 0; q < 4 * n; ++q) old[q] = obs[q];
    const double xmax = a.ox + (double)a.W * a.cs, ymax = a.oy + (double)a.H * a.cs;
    const double ro = a.r_obs, td = a.turn_dist;
    for (int i = 0; i < n; ++i) {
        double x = old[4 * i], y = old[4 * i + 1], vx = old[4 * i + 2], vy = old[4 * i + 3];
        const double aa = 0.5 * a.sigma_h * rng_normal(a.seed, trial, tick, (uint64_t)i, 0);
        const double a2 = aa * aa;
        const double c = (1.0 - a2) / (1.0 + a2), s = (2.0 * aa) / (1.0 + a2);
        const double rvx = c * vx - s * vy, rvy = s * vx + c * vy;
        vx = rvx;
        vy = rvy;
        const double lim = 2.0 * ro + td;
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            const double dx = old[4 * j] - x, dy = old[4 * j + 1] - y;
            const double d2 = dx * dx + dy * dy;
            if (d2 < lim * lim && d2 > 0.0 && dx * vx + dy * vy > 0.0) {
                const double d = sqrt(d2);
                const double nx = dx / d, ny = dy / d;
                const double vn = vx * nx + vy * ny;
                vx = vx - 2.0 * vn * nx;
                vy = vy - 2.0 * vn * ny;
                break;
            }
        }
        const double vs = sqrt(vx * vx + vy * vy);
        if (vs > 0.0) {
            const double ux = vx / vs, uy = vy / vs;
            const bool bx = sim_probe(a, mask, x, y, ux, 0.0, td);
            const bool by = sim_probe(a, mask, x, y, 0.0, uy, td);
            if (bx) vx = -vx;
            if (by) vy = -vy;
            if (!bx && !by && sim_probe(a, mask, x, y, ux, uy, td)) {
                vx = -vx;
                vy = -vy;
            }
            const double f = a.obs_speed[(int64_t)b * a.ocap + i] / vs;
            vx = vx * f;
            vy = vy * f;
        }
        x = x + vx * a.dt;
        y = y + vy * a.dt;
        if (x < a.ox + ro) { x = a.ox + ro; vx = fabs(vx); }
        if (x > xmax - ro) { x = xmax - ro; vx = -fabs(vx); }
        if (y < a.oy + ro) { y = a.oy + ro; vy = fabs(vy); }
        if (y > ymax - ro) { y = ymax - ro; vy = -fabs(vy); }
        obs[4 * i] = x;
        obs[4 * i + 1] = y;
        obs[4 * i + 2] = vx;
        obs[4 * i + 3] = vy;
    }
    // status: collision before success, then timeout
    const double x = rob[0], y = rob[1], rr = a.r_robot;
    bool coll = !(x >= a.ox && y >= a.oy && x < xmax && y < ymax);
    if (!coll) {
        const int cx0 = (int)floor((x - rr - a.ox) / a.cs), cx1 = (int)floor((x + rr - a.ox) / a.cs);
        const int cy0 = (int)floor((y - rr - a.oy) / a.cs), cy1 = (int)floor((y + rr - a.oy) / a.cs);
        for (int cy = cy0; cy <= cy1 && !coll; ++cy)
            for (int cx = cx0; cx <= cx1 && !coll; ++cx) {
                if (cx < 0 || cy < 0 || cx >= a.W || cy >= a.H) continue;
                if (!mask[(int64_t)cy * a.W + cx]) continue;
                const double ddx = (a.ox + ((double)cx + 0.5) * a.cs) - x, ddy = (a.oy + ((double)cy + 0.5) * a.cs) - y;
                if (ddx * ddx + ddy * ddy <= rr * rr) coll = true;
            }
    }
    for (int j = 0; j < n && !coll; ++j) {
        const double dx = obs[4 * j] - x, dy = obs[4 * j + 1] - y;
        const double lim = rr + ro;
        if (dx * dx + dy * dy < lim * lim) coll = true;
    }
    const int t1 = a.ticks[b] + 1;
    a.ticks[b] = t1;
    const double gx = a.goal[2 * b], gy = a.goal[2 * b + 1];
    if (coll)
        a.status[b] = 2;
    else if ((x - gx) * (x - gx) + (y - gy) * (y - gy) <= a.goal_r * a.goal_r)
        a.status[b] = 1;
    else if (t1 >= a.max_ticks)
        a.status[b] = 3;
}

// Detections of the current tick for every running trial (or only trial `only` if >= 0).
__global__ void k_sim_sense(SimArgs a, int only) {
    const int b = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if ((only >= 0 && b != only) || a.status[b] != 0 || i >= a.n_obs[b]) return;
    const double* o = a.obs + ((int64_t)b * a.ocap + i) * 4;
    const uint64_t tick = (uint64_t)a.ticks[b];
    double2 z;
    z.x = o[0] + a.sigma_z * rng_normal(a.seed, (uint64_t)b, tick, (uint64_t)i, 1);
    z.y = o[1] + a.sigma_z * rng_normal(a.seed, (uint64_t)b, tick, (uint64_t)i, 2);
    a.det[(int64_t)b * a.ocap + i] = z;
}

cudaError_t launch_sim_move(const SimArgs& a, cudaStream_t st) {
    k_sim_move<<<(a.B + 63) / 64, 64, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sim_sense(const SimArgs& a, int only, cudaStream_t st) {
    k_sim_sense<<<dim3((a.ocap + 127) / 128, a.B), 128, 0, st>>>(a, only);
    return cudaGetLastError();
}

void preload_sim_kernels() {
    cudaFuncAttributes f;
    cudaFuncGetAttributes(&f, k_sim_move);
    cudaFuncGetAttributes(&f, k_sim_sense);
    cudaGetLastError();
}

}  // namespace twg
