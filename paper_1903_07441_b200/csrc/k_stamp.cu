// k_stamp.cu -- rows a1-a3: time-warped obstacle rasterisation (Alg. 1 Map Update,
// P:679-691).
//
//   k_encode_cold     cold encode: free 0.5, static walls +0.0
//   k_unstamp         warm encode: cells stamped last tick are released as free cells that keep
//                     their value u = 0 (C7: warm start keeps every value)
//   k_goal_reset      warm encode: the previous goal cell is released as a free cell restarting at u = 0
//                     (C7: a free cell at the maximum u = 1 would be a spurious maximum)
//   k_track_predict   one thread per track, fp64: warp radius (Eq. 15 closed form, C16),
//                     warp number t (C17), horizon j (Eq. 16, C18), j Kalman predicts
//                     (Eqs. 9-10), footprint R^2 (C19-C20), bounding box
//   k_stamp           one CTA per track: cells whose centre lies within R -> obstacle,
//                     except the goal cell (warning) and the robot cell (C22)
//   k_set_goal        goal cell -> +1.0 (u = 1, phi = 0)
//
// Bit-exactness with oracle/twg_oracle.c (orc_classify): every fp64 expression is
// the same IEEE operation sequence (library compiled with -fmad=false); cos/sin of
// theta come from the host libm (C25); llround = round half away from zero.
#include "twg_kernels.cuh"

namespace twg {

__global__ void k_encode_cold(EncodeArgs e) {
    pdl_enter();
    const ScenParams& sp = e.params[blockIdx.z];
    if (sp.warm) return;
    const int b = sp.b;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x == 0 && y == 0) e.fixbox[2 * b + 1] = make_int4(1, 0, 1, 0);  // no imported fixed values left
    if (y >= e.H || x >= e.P) return;
    float v = 0.0f;  // pad columns: fixed obstacle
    if (x < e.W) v = e.mask[((int64_t)b * e.H + y) * e.W + x] ? 0.0f : -0.5f;
    (sp.cur ? e.u1 : e.u0)[(int64_t)b * e.sstride + (int64_t)y * e.P + x] = v;
}

__global__ void k_unstamp(EncodeArgs e) {
    pdl_enter();
    const ScenParams& sp = e.params[blockIdx.y];
    if (!sp.warm || (int)blockIdx.x >= sp.n_prev_boxes) return;
    const int b = sp.b;
    const int4 bx = e.boxes[(int64_t)b * e.cap + blockIdx.x];  // (x0, x1, y0, y1)
    if (bx.x > bx.y || bx.z > bx.w) return;
    const int nx = bx.y - bx.x + 1, n = nx * (bx.w - bx.z + 1);
    float* f = (sp.cur ? e.u1 : e.u0) + (int64_t)b * e.sstride;
    const uint8_t* m = e.mask + (int64_t)b * e.H * e.W;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const int x = bx.x + q % nx, y = bx.z + q / nx;
        TWG_CHECK(x >= 0 && x < e.W && y >= 0 && y < e.H);
        float* p = f + (int64_t)y * e.P + x;
        if (__float_as_uint(*p) == 0u && m[(int64_t)y * e.W + x] == 0) *p = -0.0f;  // free, u = 0
    }
}

__device__ __forceinline__ void goal_reset_one(const EncodeArgs& e, const ScenParams& sp) {
    e.flags[sp.b] = 0;  // warning flags of this call (set by k_stamp, which runs after)
    if (!sp.warm || sp.old_gx < 0 || sp.old_gy < 0 || sp.old_gy >= e.H) return;
    if (sp.old_gx == sp.gx && sp.old_gy == sp.gy) return;
    const int b = sp.b;
    if (e.mask[((int64_t)b * e.H + sp.old_gy) * e.W + sp.old_gx]) return;
    (sp.cur ? e.u1 : e.u0)[(int64_t)b * e.sstride + (int64_t)sp.old_gy * e.P + sp.old_gx] = -0.0f;  // free, u = 0
}

__device__ __forceinline__ void set_goal_one(const EncodeArgs& e, const ScenParams& sp) {
    const bool in = sp.gy >= 0 && sp.gy < e.H;  // else the goal lies in another row slab
    // the goal is the field's positive fixed cell: its box keeps k_rb_tblock's nearby warps on the
    // scalar path
    e.fixbox[2 * sp.b] = in ? make_int4(sp.gx, sp.gx, sp.gy, sp.gy) : make_int4(1, 0, 1, 0);
    if (!in) return;
    (sp.cur ? e.u1 : e.u0)[(int64_t)sp.b * e.sstride + (int64_t)sp.gy * e.P + sp.gx] = 1.0f;
}

// Standalone launches for encodes without tracks; with tracks, k_track_predict resets the goal and
// k_stamp sets it (one thread of the scenario's first CTA each).
__global__ void k_goal_reset(EncodeArgs e) {
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= e.nscen) return;
    goal_reset_one(e, e.params[k]);
}

// Round half away from zero of a non-negative double (C25; equals llround for x >= 0).
__device__ __forceinline__ long long round_half_away(double x) {
    if (!(x < 4.0e18)) return 4000000000000000000LL;  // far beyond any horizon clamp
    const double t = trunc(x);
    return (long long)t + ((x - t) >= 0.5 ? 1 : 0);
}

__global__ void k_track_predict(EncodeArgs e) {
    pdl_enter();
    const ScenParams& sp = e.params[blockIdx.y];
    if (blockIdx.x == 0 && threadIdx.x == 0) goal_reset_one(e, sp);  // before k_stamp (next launch)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= sp.n_tracks) return;
    const int b = sp.b;
    const int64_t slot = (int64_t)b * e.cap + i;
    twg_track tr;
    if (e.src) {  // caller-supplied tracks replace the resident table (f1); copied here, no scatter pass
        tr = e.src[sp.track_off + i];
        e.tracks[slot] = tr;
        e.missed[slot] = 0;
    } else {
        tr = e.tracks[slot];
    }
    const WarpCfgDev& w = *e.wcfg;
    // a1: warp radius (Eq. 15 with the P:463-465 centre, closed form C16) from x_hat (C24)
    const double dx = tr.x[0] - sp.xr;
    const double dy = tr.x[1] - sp.yr;
    const double aa = sp.c * dx + sp.s * dy;
    const double bb = sp.s * dx - sp.c * dy;
    const double rx = (sqrt(4.0 * aa * aa + 12.16 * bb * bb) - 1.8 * aa) / 0.38;
    double tf = ceil(rx / w.w);
    if (tf < 1.0) tf = 1.0;
    const int t = (int)tf;
    long long jl;
    if (w.hmode == 0) {
        // a2: horizon j = clamp(round(v t), 0, hmax), v = speed_r / max(|v_hat|, eps_v) (Eq. 16, C18)
        double so = sqrt(tr.x[2] * tr.x[2] + tr.x[3] * tr.x[3]);
        if (so < w.eps_v) so = w.eps_v;
        const double v = sp.speed / so;
        jl = round_half_away(v * (double)t);
    } else if (!(sp.speed > 0.0)) {
        jl = w.hmax;  // robot at rest never reaches the ring (C26)
    } else {
        // ring time: j = round(t w / (speed_r dt)) (C26)
        const double steps = ((double)t * w.w) / (sp.speed * w.dt);
        jl = steps < 0.0 ? -round_half_away(-steps) : round_half_away(steps);
    }
    if (jl < 0) jl = 0;
    if (jl > w.hmax) jl = w.hmax;
    const int j = (int)jl;
    // j x (x <- A x; P <- A P A^T + Q)  (Eqs. 9-10, A of P:548-553), dense, k ascending
    double A[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) A[q] = 0.0;
    A[0] = 1.0; A[5] = 1.0; A[10] = 1.0; A[15] = 1.0;
    A[2] = w.dt; A[7] = w.dt;
    double xc[4], Pc[16], AP[16], xn[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) xc[q] = tr.x[q];
#pragma unroll
    for (int q = 0; q < 16; ++q) Pc[q] = tr.P[q];
    for (int step = 0; step < j; ++step) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + A[r * 4 + k] * xc[k];
            xn[r] = acc;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) xc[r] = xn[r];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int col = 0; col < 4; ++col) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) acc = acc + A[r * 4 + k] * Pc[k * 4 + col];
                AP[r * 4 + col] = acc;
            }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int col = 0; col < 4; ++col) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) acc = acc + AP[r * 4 + k] * A[col * 4 + k];
                Pc[r * 4 + col] = acc + w.Q[r * 4 + col];
            }
    }
    // footprint: sigma^2 = (P00 + P11) / 2 of the predicted (C19) or posterior (C27) covariance;
    // Gaussian >= 1/2 <=> d^2 <= 2 ln2 sigma^2; U safety disk (C20)
    const double sig2 = w.fmode == 0 ? (Pc[0] + Pc[5]) * 0.5 : (tr.P[0] + tr.P[5]) * 0.5;
    const double g = 1.3862943611198906 * sig2;
    const double s2 = w.rs * w.rs;
    const double R2 = g > s2 ? g : s2;
    e.t_out[slot] = t;
    e.j_out[slot] = j;
    e.pred[slot * 3 + 0] = xc[0];
    e.pred[slot * 3 + 1] = xc[1];
    e.pred[slot * 3 + 2] = R2;
    // bounding box of the disk, one cell of margin (any superset gives the same cell set)
    const double R = sqrt(R2);
    const double lx = floor((xc[0] - R - e.ox) / e.cs) - 1.0, hx = ceil((xc[0] + R - e.ox) / e.cs) + 1.0;
    const double ly = floor((xc[1] - R - e.oy) / e.cs) - 1.0, hy = ceil((xc[1] + R - e.oy) / e.cs) + 1.0;
    int4 box = make_int4(1, 0, 1, 0);  // empty
    if (!(hx < 0.0 || hy < 0.0 || lx > (double)(e.W - 1) || ly > (double)(e.H - 1))) {
        box.x = lx < 0.0 ? 0 : (int)lx;
        box.y = hx > (double)(e.W - 1) ? e.W - 1 : (int)hx;
        box.z = ly < 0.0 ? 0 : (int)ly;
        box.w = hy > (double)(e.H - 1) ? e.H - 1 : (int)hy;
    }
    e.boxes[slot] = box;
}

__global__ void k_stamp(EncodeArgs e) {
    pdl_enter();
    const ScenParams& sp = e.params[blockIdx.y];
    if (blockIdx.x == 0 && threadIdx.x == 0) set_goal_one(e, sp);  // k_stamp never writes the goal cell
    if ((int)blockIdx.x >= sp.n_tracks) return;
    const int b = sp.b;
    const int64_t slot = (int64_t)b * e.cap + blockIdx.x;
    const int4 bx = e.boxes[slot];
    if (bx.x > bx.y || bx.z > bx.w) return;
    const double xp = e.pred[slot * 3 + 0], yp = e.pred[slot * 3 + 1], R2 = e.pred[slot * 3 + 2];
    const int nx = bx.y - bx.x + 1, n = nx * (bx.w - bx.z + 1);
    float* f = (sp.cur ? e.u1 : e.u0) + (int64_t)b * e.sstride;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const int i = bx.x + q % nx, k = bx.z + q / nx;
        const double cx = e.ox + ((double)i + 0.5) * e.cs;
        const double cy = e.oy + ((double)k + 0.5) * e.cs;
        const double ddx = cx - xp, ddy = cy - yp;
        if (ddx * ddx + ddy * ddy <= R2) {
            TWG_CHECK(i >= 0 && i < e.W && k >= 0 && k < e.H);
            if (i == sp.gx && k == sp.gy) {
                atomicOr(&e.flags[b], 1);  // TWG_W_GOAL_SWALLOWED: the goal is kept
            } else if (!(i == sp.rcx && k == sp.rcy)) {
                f[(int64_t)k * e.P + i] = 0.0f;  // obstacle (idempotent; overlapping disks race benignly)
            }
        }
    }
}

__global__ void k_set_goal(EncodeArgs e) {
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= e.nscen) return;
    set_goal_one(e, e.params[k]);
}


// Fresh context: every cell free at 0.5, pad columns fixed obstacles.
__global__ void k_init_field(float* __restrict__ u, int64_t P, int64_t sstride, int W, int H) {
    const int b = blockIdx.z;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (y >= H || x >= P) return;
    u[(int64_t)b * sstride + (int64_t)y * P + x] = x < W ? -0.5f : 0.0f;
}

cudaError_t launch_init_field(float* u, int64_t P, int64_t sstride, int W, int H, int B, cudaStream_t st) {
    dim3 blk(128, 4);
    dim3 grid((unsigned)((P + 127) / 128), (H + 3) / 4, B);
    k_init_field<<<grid, blk, 0, st>>>(u, P, sstride, W, H);
    return cudaGetLastError();
}

// Field export (twg_get_field): mode 0 raw, 1 |u|, 2 phi = 1 - |u|; pitched -> dense.
__global__ void k_convert(const float* __restrict__ src, int64_t P, int W, int H, float* __restrict__ dst, int mode) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= W || y >= H) return;
    const float v = src[(int64_t)y * P + x];
    dst[(int64_t)y * W + x] = mode == 0 ? v : (mode == 1 ? fabsf(v) : 1.0f - fabsf(v));
}

// Field import (twg_set_field): dense raw -> pitched, pad columns +0.0; the bounding box of the
// positive cells (fixed cells with u > 0, e.g. the goal or Dirichlet test data) is accumulated into
// box (x0, x1, y0, y1), which the caller set empty.
__global__ void k_import(const float* __restrict__ src, int W, int H, float* __restrict__ dst, int64_t P,
                         int4* __restrict__ box) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= P || y >= H) return;
    const float v = x < W ? src[(int64_t)y * W + x] : 0.0f;
    dst[(int64_t)y * P + x] = v;
    if (__float_as_int(v) > 0) {
        int* b = reinterpret_cast<int*>(box);
        atomicMin(b + 0, x);
        atomicMax(b + 1, x);
        atomicMin(b + 2, y);
        atomicMax(b + 3, y);
    }
}

cudaError_t launch_convert(const float* src, int64_t P, int W, int H, float* dst, int mode, cudaStream_t st) {
    dim3 blk(128, 4);
    dim3 grid((W + 127) / 128, (H + 3) / 4);
    k_convert<<<grid, blk, 0, st>>>(src, P, W, H, dst, mode);
    return cudaGetLastError();
}

cudaError_t launch_import(const float* src, int W, int H, float* dst, int64_t P, int4* box, cudaStream_t st) {
    dim3 blk(128, 4);
    dim3 grid((unsigned)((P + 127) / 128), (H + 3) / 4);
    k_import<<<grid, blk, 0, st>>>(src, W, H, dst, P, box);
    return cudaGetLastError();
}


__global__ void k_warp_map(int32_t* __restrict__ out, int W, int H, double cs, double ox, double oy, double xr,
                           double yr, double c, double s, double w);

void preload_stamp_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_warp_map);
    cudaFuncGetAttributes(&a, k_encode_cold);
    cudaFuncGetAttributes(&a, k_unstamp);
    cudaFuncGetAttributes(&a, k_goal_reset);
    cudaFuncGetAttributes(&a, k_track_predict);
    cudaFuncGetAttributes(&a, k_stamp);
    cudaFuncGetAttributes(&a, k_set_goal);
    cudaFuncGetAttributes(&a, k_convert);
    cudaFuncGetAttributes(&a, k_import);
    cudaGetLastError();
}

// Threads per footprint CTA of k_unstamp / k_stamp: a few scenarios (C3: 200 tracks, a fresh track's
// footprint ~1850 cells) fill the GPU only with wide CTAs; a batch (C5: 1024 x 20 footprints of ~120
// cells, the CTA loops over its box) with narrow ones -- 1024-thread CTAs there mostly idle.
static int box_threads(int nscen, int wide) { return nscen > 8 ? 128 : wide; }

cudaError_t launch_encode(const EncodeArgs& e, int max_prev_boxes, int max_tracks, int any_cold, int* n_launch,
                          cudaStream_t st) {
    int nl = 0;
    if (any_cold) {
        dim3 blk(128, 4);
        dim3 grid((unsigned)((e.P + 127) / 128), (e.H + 3) / 4, e.nscen);
        if (cudaError_t err = launch_pdl(k_encode_cold, grid, blk, 0, st, e)) return err;
        ++nl;
    }
    if (max_prev_boxes > 0) {
        if (cudaError_t err = launch_pdl(k_unstamp, dim3(max_prev_boxes, e.nscen), dim3(box_threads(e.nscen, 1024)), 0, st, e)) return err;
        ++nl;
    }
    const int sb = (e.nscen + 127) / 128;
    if (max_tracks > 0) {  // the goal reset / set ride on the first CTA of each scenario
        if (cudaError_t err = launch_pdl(k_track_predict, dim3((max_tracks + 63) / 64, e.nscen), dim3(64), 0, st, e))
            return err;
        if (cudaError_t err = launch_pdl(k_stamp, dim3(max_tracks, e.nscen), dim3(box_threads(e.nscen, 512)), 0, st, e)) return err;
        nl += 2;
    } else {
        if (cudaError_t err = launch_pdl(k_goal_reset, dim3(sb), dim3(128), 0, st, e)) return err;
        if (cudaError_t err = launch_pdl(k_set_goal, dim3(sb), dim3(128), 0, st, e)) return err;
        nl += 2;
    }
    if (n_launch) *n_launch = nl;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ per-cell warp map (f3)
// The paper's kernel 1 ("calculate the warp of each cell"): t = max(1, ceil(r_x / w)) of an
// obstacle at each cell centre, r_x the Eq. 15 closed form (C16) -- the same fp64 sequence as
// k_track_predict.  out: [H][W] int32.
__global__ void k_warp_map(int32_t* __restrict__ out, int W, int H, double cs, double ox, double oy, double xr,
                           double yr, double c, double s, double w) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= W) return;
    const double px = ox + ((double)x + 0.5) * cs;
    const double py = oy + ((double)y + 0.5) * cs;
    const double dx = px - xr, dy = py - yr;
    const double aa = c * dx + s * dy;
    const double bb = s * dx - c * dy;
    const double rx = (sqrt(4.0 * aa * aa + 12.16 * bb * bb) - 1.8 * aa) / 0.38;
    double tf = ceil(rx / w);
    if (tf < 1.0) tf = 1.0;
    out[(int64_t)y * W + x] = (int32_t)tf;
}

cudaError_t launch_warp_map(int32_t* out, int W, int H, double cs, double ox, double oy, double xr, double yr, double c,
                            double s, double w, cudaStream_t st) {
    k_warp_map<<<dim3((W + 255) / 256, H), 256, 0, st>>>(out, W, H, cs, ox, oy, xr, yr, c, s, w);
    return cudaGetLastError();
}

}  // namespace twg
