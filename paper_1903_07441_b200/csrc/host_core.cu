// host_core.cu -- host side of the C ABI shared by every entry point: validation, error
// reporting, pinned staging, buffer management and the orchestration of rows a1-a9 (encode, relax,
// path).  Every step of the hot path runs in the kernels of k_stamp.cu (a1-a3), k_relax.cu (a4-a6)
// and k_path.cu (a7-a9); the entry points themselves are in api*.cu.
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "api_host.cuh"

namespace twg {
namespace host {

std::string g_create_err;  // message of the last failed twg_create

twg_status fail(twg_ctx* c, twg_status st, const std::string& msg) {
    if (c) c->err = msg;
    else g_create_err = msg;
    return st;
}


bool is_device_ptr(const void* p) {
    if (p == nullptr) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3D map {W, H, B} over one ping-pong buffer; box {128, rows, 1}; OOB -> zero fill.
bool make_tmap(CUtensorMap* m, float* base, int W, int H, int B, int64_t P, int rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)(P * 4), (cuuint64_t)(P * 4 * (int64_t)H)};
    cuuint32_t box[3] = {(cuuint32_t)kStripW, (cuuint32_t)rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The index matrix as a 2D {P, H * B} uint16 tensor with box {256, 176}: one box lands in shared
// memory as 176 rows of 256 contiguous descriptors (k_walk windows, row pitch 256).
bool make_dir_map(CUtensorMap* m, uint8_t* base, int H, int B, int64_t P) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)H * (cuuint64_t)B};
    cuuint64_t strides[1] = {(cuuint64_t)P};
    cuuint32_t box[2] = {256, 176};  // may exceed P: out-of-range columns are zero-filled
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}


// Pinned host staging ring.  Regions are handed out in order; when the ring wraps
// (or must grow) the stream is synchronised first, so a region is never rewritten
// while an earlier asynchronous copy may still read it.
cudaError_t stage_alloc(twg_ctx* c, size_t bytes, void** out) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes > c->h_stage_bytes) {
        cudaError_t e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) return e;
        if (c->h_stage) cudaFreeHost(c->h_stage);
        c->h_stage = nullptr;
        c->h_stage_bytes = 0;
        const size_t nb = std::max<size_t>(bytes, size_t(8) << 20);
        e = cudaMallocHost(&c->h_stage, nb);
        if (e != cudaSuccess) return e;
        c->h_stage_bytes = nb;
        c->stage_off = 0;
    } else if (c->stage_off + bytes > c->h_stage_bytes) {
        cudaError_t e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) return e;
        c->stage_off = 0;
    }
    *out = static_cast<char*>(c->h_stage) + c->stage_off;
    c->stage_off += bytes;
    return cudaSuccess;
}

// Grow the per-scenario track arrays to `cap` entries, keeping their contents.
twg_status ensure_track_cap(twg_ctx* c, int cap) {
    if (cap <= c->track_cap) return TWG_OK;
    int nc = std::max(cap, std::max(2 * c->track_cap, 64));
    const size_t B = c->B;
    twg_track* t0;
    int *t1, *t2;
    double* t3;
    int4* t4;
    int* t5;
    TWG_CUDA(c, dev_alloc(&t0, B * nc));
    TWG_CUDA(c, dev_alloc(&t5, B * nc));
    TWG_CUDA(c, dev_alloc(&t1, B * nc));
    TWG_CUDA(c, dev_alloc(&t2, B * nc));
    TWG_CUDA(c, dev_alloc(&t3, B * nc * 3));
    TWG_CUDA(c, dev_alloc(&t4, B * nc));
    if (c->track_cap > 0) {
        const int oc = c->track_cap;
        TWG_CUDA(c, cudaMemcpy2DAsync(t0, nc * sizeof(twg_track), c->d_tracks, oc * sizeof(twg_track),
                                      oc * sizeof(twg_track), B, cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaMemcpy2DAsync(t1, nc * sizeof(int), c->d_t, oc * sizeof(int), oc * sizeof(int), B,
                                      cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaMemcpy2DAsync(t2, nc * sizeof(int), c->d_j, oc * sizeof(int), oc * sizeof(int), B,
                                      cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaMemcpy2DAsync(t3, nc * 3 * sizeof(double), c->d_pred, oc * 3 * sizeof(double),
                                      oc * 3 * sizeof(double), B, cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaMemcpy2DAsync(t4, nc * sizeof(int4), c->d_boxes, oc * sizeof(int4), oc * sizeof(int4), B,
                                      cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaMemcpy2DAsync(t5, nc * sizeof(int), c->d_missed, oc * sizeof(int), oc * sizeof(int), B,
                                      cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaStreamSynchronize(c->stream));
        cudaFree(c->d_tracks);
        cudaFree(c->d_t);
        cudaFree(c->d_j);
        cudaFree(c->d_pred);
        cudaFree(c->d_boxes);
        cudaFree(c->d_missed);
    }
    c->d_tracks = t0;
    c->d_t = t1;
    c->d_j = t2;
    c->d_pred = t3;
    c->d_boxes = t4;
    c->d_missed = t5;
    c->track_cap = nc;
    return TWG_OK;
}

// Parameter block: [WarpCfgDev | pad to 256 B | ScenParams x n], so one copy uploads both.
constexpr size_t kParamOff = 256;
static_assert(sizeof(WarpCfgDev) <= kParamOff, "warp cfg does not fit the parameter block header");
twg_status ensure_params(twg_ctx* c, int n) {
    if (n <= c->params_cap && c->d_param_block) return TWG_OK;
    if (c->d_param_block) cudaFree(c->d_param_block);
    c->d_param_block = nullptr;
    c->d_params = nullptr;
    c->d_wcfg = nullptr;
    const int nc = std::max(n, 1);
    TWG_CUDA(c, dev_alloc(&c->d_param_block, kParamOff + (size_t)nc * sizeof(ScenParams)));
    c->d_wcfg = reinterpret_cast<WarpCfgDev*>(c->d_param_block);
    c->d_params = reinterpret_cast<ScenParams*>(c->d_param_block + kParamOff);
    c->params_cap = nc;
    return TWG_OK;
}

twg_status ensure_path_cap(twg_ctx* c, int max_len, int max_smooth) {
    const size_t B = c->B;
    if (max_len > c->path_len_cap) {
        int nc = std::max(max_len, 256);
        if (c->d_cells) cudaFree(c->d_cells);
        if (c->d_wp) cudaFree(c->d_wp);
        c->d_cells = nullptr;
        c->d_wp = nullptr;
        TWG_CUDA(c, dev_alloc(&c->d_cells, B * nc));
        TWG_CUDA(c, dev_alloc(&c->d_wp, B * nc));
        c->path_len_cap = nc;
        if (B <= (size_t)kSpecMaxB) {
            if (c->d_seg_cells) cudaFree(c->d_seg_cells);
            c->d_seg_cells = nullptr;
            TWG_CUDA(c, dev_alloc(&c->d_seg_cells, B * kSpecMax * (size_t)(nc + 1)));
            if (!c->d_spec) {  // no markers before the first walk
                TWG_CUDA(c, dev_alloc(&c->d_spec, B));
                TWG_CUDA(c, cudaMemsetAsync(c->d_spec, 0, B * sizeof(SpecTab), c->stream));
            }
            if (!c->d_seg) TWG_CUDA(c, dev_alloc(&c->d_seg, B * (kSpecMax + 1)));
        }
    }
    if (max_smooth > c->smooth_cap) {
        int nc = std::max(max_smooth, 256);
        if (c->d_smooth) cudaFree(c->d_smooth);
        c->d_smooth = nullptr;
        TWG_CUDA(c, dev_alloc(&c->d_smooth, B * nc));
        c->smooth_cap = nc;
    }
    return TWG_OK;
}

twg_status check_ctx(twg_ctx* c) {
    if (!c) return TWG_E_INVALID_ARG;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, TWG_E_CUDA, cudaGetErrorString(e));
    return TWG_OK;
}

// One scenario's encode request.

// Host validation -> robot cell.
twg_status validate(twg_ctx* c, const EncodeReq& r, int* rcx, int* rcy) {
    const bool slab = c->ghost > 0;  // goal and robot may belong to another slab
    const bool g_in = r.gx >= 0 && r.gy >= 0 && r.gx < c->W && r.gy < c->H;
    if (!g_in && !(slab && r.gx >= 0 && r.gx < c->W))
        return fail(c, TWG_E_OUT_OF_BOUNDS, "goal cell outside the grid");
    const uint8_t* m = c->hmask.data() + (size_t)r.b * c->H * c->W;
    if (g_in && m[(size_t)r.gy * c->W + r.gx]) return fail(c, TWG_E_OVERLAPPING_CLASSES, "goal cell on a static wall");
    const double fx = std::floor((r.robot.x - c->ox) / c->cs), fy = std::floor((r.robot.y - c->oy) / c->cs);
    const bool r_in = fx >= 0.0 && fy >= 0.0 && fx < (double)c->W && fy < (double)c->H;
    if (!r_in && !slab) return fail(c, TWG_E_OUT_OF_BOUNDS, "robot cell outside the grid");
    *rcx = r_in ? (int)fx : -1;
    *rcy = r_in ? (int)fy : -1;
    if (r_in && m[(size_t)*rcy * c->W + *rcx]) return fail(c, TWG_E_INVALID_START, "robot cell on a static wall");
    if (r.n < 0) return fail(c, TWG_E_INVALID_ARG, "negative track count");
    return TWG_OK;
}

// Rows a1-a3 for a list of scenarios.  tracks: concatenated per request (host or device).
// resident: use the tracker tables (row f1) already in d_tracks instead of caller tracks.
twg_status encode(twg_ctx* c, const std::vector<EncodeReq>& reqs, const twg_track* tracks, const twg_warp_cfg* wc,
                  int warm_req, bool resident) {
    if (!wc) return fail(c, TWG_E_INVALID_ARG, "null warp cfg");
    if ((wc->horizon_mode != 0 && wc->horizon_mode != 1) || (wc->footprint_mode != 0 && wc->footprint_mode != 1))
        return fail(c, TWG_E_INVALID_ARG, "horizon_mode / footprint_mode must be 0 or 1");
    const int ns = (int)reqs.size();
    std::vector<ScenParams> ps(ns);
    int max_n = 0, max_prev = 0, any_cold = 0;
    int64_t total = 0;
    for (int k = 0; k < ns; ++k) {
        const EncodeReq& r = reqs[k];
        int rcx, rcy;
        twg_status st = validate(c, r, &rcx, &rcy);
        if (st != TWG_OK) return st;
        twg_ctx::Scen& sc = c->scen[r.b];
        ScenParams& p = ps[k];
        p.xr = r.robot.x;
        p.yr = r.robot.y;
        p.c = std::cos(r.robot.theta);  // host libm (C25)
        p.s = std::sin(r.robot.theta);
        p.speed = r.robot.speed;
        p.b = r.b;
        p.gx = r.gx;
        p.gy = r.gy;
        p.rcx = rcx;
        p.rcy = rcy;
        const bool warm = warm_req && sc.encoded && !sc.static_dirty;
        p.warm = warm ? 1 : 0;
        p.old_gx = warm ? sc.gx : -1;
        p.old_gy = warm ? sc.gy : -1;
        p.cur = c->cur[r.b];
        p.n_tracks = r.n;
        p.n_prev_boxes = warm ? sc.n_boxes : 0;
        max_n = std::max(max_n, r.n);
        max_prev = std::max(max_prev, p.n_prev_boxes);
        any_cold |= !warm;
        total += r.n;
    }
    twg_status st = ensure_track_cap(c, std::max(max_n, 1));
    if (st != TWG_OK) return st;
    st = ensure_params(c, ns);
    if (st != TWG_OK) return st;
    // caller tracks: device input is read in place, host input goes through the pinned staging ring
    // in one H2D copy; k_track_predict copies them into the [B][cap] resident table as it reads them
    const twg_track* src = nullptr;
    if (total > 0 && !resident) {
        src = tracks;
        if (!is_device_ptr(tracks)) {
            if (c->track_tmp_cap < total) {
                if (c->d_track_tmp) cudaFree(c->d_track_tmp);
                c->d_track_tmp = nullptr;
                TWG_CUDA(c, dev_alloc(&c->d_track_tmp, (size_t)total));
                c->track_tmp_cap = total;
            }
            twg_track* ht = nullptr;
            TWG_CUDA(c, stage_alloc(c, (size_t)total * sizeof(twg_track), reinterpret_cast<void**>(&ht)));
            int64_t first = reqs[0].track_off;
            std::memcpy(ht, tracks + first, (size_t)total * sizeof(twg_track));
            TWG_CUDA(c, cudaMemcpyAsync(c->d_track_tmp, ht, (size_t)total * sizeof(twg_track), cudaMemcpyHostToDevice,
                                        c->stream));
            src = c->d_track_tmp - first;  // offsets below are relative to the caller's array
        }
        for (int k = 0; k < ns; ++k) ps[k].track_off = reqs[k].track_off;
    }
    // per-scenario params + cfg (pinned staging, one copy each)
    WarpCfgDev w;
    w.dt = wc->dt;
    std::memcpy(w.Q, wc->Q, sizeof(w.Q));
    w.w = wc->warp_spacing;
    w.eps_v = wc->eps_v;
    w.rs = wc->safety_radius;
    w.hmax = wc->horizon_max;
    w.hmode = wc->horizon_mode;
    w.fmode = wc->footprint_mode;
    // warp cfg + per-scenario params: one copy into the parameter block (warning flags are cleared
    // by k_goal_reset, which runs before the stamping kernels that set them)
    const size_t pbytes = kParamOff + ns * sizeof(ScenParams);
    char* hs = nullptr;
    TWG_CUDA(c, stage_alloc(c, pbytes, reinterpret_cast<void**>(&hs)));
    std::memcpy(hs, &w, sizeof(w));
    std::memcpy(hs + kParamOff, ps.data(), ns * sizeof(ScenParams));
    TWG_CUDA(c, cudaMemcpyAsync(c->d_param_block, hs, pbytes, cudaMemcpyHostToDevice, c->stream));
    EncodeArgs e;
    e.u0 = c->u[0];
    e.u1 = c->u[1];
    e.P = c->P;
    e.sstride = c->sstride;
    e.W = c->W;
    e.H = c->H;
    e.mask = c->mask;
    e.params = c->d_params;
    e.nscen = ns;
    e.wcfg = c->d_wcfg;
    e.tracks = c->d_tracks;
    e.src = src;
    e.missed = c->d_missed;
    e.cap = c->track_cap;
    e.t_out = c->d_t;
    e.j_out = c->d_j;
    e.pred = c->d_pred;
    e.boxes = c->d_boxes;
    e.flags = c->d_flags;
    e.fixbox = c->d_fixbox;
    e.cs = c->cs;
    e.ox = c->ox;
    e.oy = c->oy;
    int nl = 0;
    TWG_CUDA(c, launch_encode(e, max_prev, max_n, any_cold, &nl, c->stream));
    c->launches += nl;
    // host-side bookkeeping for the next warm encode
    for (int k = 0; k < ns; ++k) {
        twg_ctx::Scen& sc = c->scen[reqs[k].b];
        sc.gx = ps[k].gx;
        sc.gy = ps[k].gy;
        sc.rcx = ps[k].rcx;
        sc.rcy = ps[k].rcy;
        sc.rx = reqs[k].robot.x;
        sc.ry = reqs[k].robot.y;
        sc.n_tracks = reqs[k].n;
        if (!resident) sc.trk_n = reqs[k].n;
        sc.n_boxes = reqs[k].n;
        sc.encoded = true;
        sc.static_dirty = false;
    }
    return TWG_OK;
}

// Output rows per warp (hseg).  hseg + 4T is a multiple of NW = 2T + 2 (the kernel streams whole
// NW-row blocks, so any other value pays for padded rows) and even (the colour parity of the first
// row is a compile-time constant).  Among those, pick the one minimising the load model measured on
// B200: the CTAs run in waves of the kernel's occupancy (CTAs resident per
// SM), and a wave of n CTAs takes ~ (hseg + 4T) x max(1, n warps / 8) -- throughput saturates at eight
// warps per SM (one 8-warp CTA at T = 6, 198 registers).
int auto_hseg(int T, int H, int n_strips, int nscen, int cfg_rows, int n_sm) {
    const int NW = 2 * T + 2;
    if (cfg_rows > 0) {
        int h = std::min(cfg_rows, H);
        h = (h + 1) & ~1;
        return std::max(h, 2);
    }
    const int resident = std::max(1, rb_tblock_ctas_per_sm(T));
    int best_h = 2;
    double best = 1e300;
    for (int k = 1; k <= 256; ++k) {
        const int h = k * NW - 4 * T;
        if (h < 2) continue;
        const int hh = std::min(h, (H + 1) & ~1);
        const long long segs = (H + hh - 1) / hh;
        const long long ctas = (segs * n_strips * nscen + kWarpsPerCta - 1) / kWarpsPerCta;
        const long long per_sm = (ctas + n_sm - 1) / n_sm;
        double cost = 0.0;
        for (long long left = per_sm; left > 0; left -= resident)
            cost += (double)(hh + 4 * T) * std::max(1.0, (double)std::min<long long>(left, resident) * kWarpsPerCta / 8.0);
        if (cost < best * 0.999) {
            best = cost;
            best_h = hh;
        }
        if (h >= H) break;
    }
    return std::max(best_h, 2);
}

// Task lists and counters of the lexicographic mode: 32 x 32 tiles, tasks (sweep s, tile (i, j)) of
// one launch of `sweeps` sweeps ordered by wavefront time i + j + 2 s, then s, then j.  Every
// dependency of a task has a smaller time, so the order is topological.  Lists are cached per
// launch length (a relaxation uses at most two: kLexMaxSweeps and its remainder).
constexpr int kLexMaxSweeps = 64;  // sweeps per persistent launch
int2* lex_tasks(twg_ctx* c, int sweeps) {
    for (auto& e : c->lex_lists)
        if (e.first == sweeps) return e.second;
    const int tx = c->lex_tx, ty = c->lex_ty;
    std::vector<int2> ord;
    ord.reserve((size_t)tx * ty * sweeps);
    const int dmax = tx + ty - 2;
    for (int tau = 0; tau <= dmax + 2 * (sweeps - 1); ++tau)
        for (int s = 0; s < sweeps; ++s) {
            const int d = tau - 2 * s;
            if (d < 0 || d > dmax) continue;
            for (int j = 0; j < ty; ++j) {
                const int i = d - j;
                if (i >= 0 && i < tx) ord.push_back(make_int2(i | (s << 16), j));
            }
        }
    int2* d = nullptr;
    if (dev_alloc(&d, ord.size()) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, ord.data(), ord.size() * sizeof(int2), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    if (c->lex_lists.size() >= 4) {  // keep a handful
        cudaFree(c->lex_lists.front().second);
        c->lex_lists.erase(c->lex_lists.begin());
    }
    c->lex_lists.emplace_back(sweeps, d);
    return d;
}

twg_status ensure_lex(twg_ctx* c) {
    if (c->d_lex_tdone) return TWG_OK;
    c->lex_tx = (c->W + 31) / 32;
    c->lex_ty = (c->H + 31) / 32;
    TWG_CUDA(c, dev_alloc(&c->d_lex_tdone, (size_t)c->B * c->lex_tx * c->lex_ty));
    TWG_CUDA(c, dev_alloc(&c->d_lex_task, 1));
    return TWG_OK;
}

// ---------------------------------------------------------------- rows a4-a6
// One red-black tile launch of t sweeps over output rows [lo, hi) of every participating scenario
// of c.  The colour parity of row lo is folded into the kernel's compile-time parity (QOFF).
static twg_status launch_rb_range(twg_ctx* c, const twg_relax_cfg* cfg, int t, int lp, int lo, int hi, bool resid,
                                  int nscen, cudaStream_t st) {
    RelaxArgs a;
    a.u0 = c->u[0];
    a.u1 = c->u[1];
    a.cur = c->d_cur;
    a.P = c->P;
    a.sstride = c->sstride;
    a.W = c->W;
    a.H = c->H;
    a.done = c->d_done;
    a.res = c->d_res_bits;
    a.res_r0 = c->ghost;
    a.res_r1 = c->H - c->ghost;
    a.lp = lp & 1;
    a.fixbox = c->d_fixbox;
    // TWG_RELAX_SLOW=1: every warp on the scalar path (tests); =2: no warp (timing experiments only --
    // wrong results near positive fixed cells)
    static const int force_slow = [] { const char* e = std::getenv("TWG_RELAX_SLOW"); return e ? std::atoi(e) : 0; }();
    a.force_slow = force_slow;
    a.row_lo = lo;
    a.row_hi = hi;
    a.n_strips = (c->W + out_cols(t) - 1) / out_cols(t);
    a.hseg = auto_hseg(t, hi - lo, a.n_strips, std::max(nscen, 1), cfg->rows_per_warp, c->n_sm);
    a.seg_begin = 0;
    a.seg_end = (hi - lo + a.hseg - 1) / a.hseg;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool prof = c->prof && st == c->stream;
    if (prof) {
        while ((int)c->ev_pool.size() < c->ev_used + 2) {
            cudaEvent_t ev;
            TWG_CUDA(c, cudaEventCreate(&ev));
            c->ev_pool.push_back(ev);
        }
        e0 = c->ev_pool[c->ev_used++];
        e1 = c->ev_pool[c->ev_used++];
        TWG_CUDA(c, cudaEventRecord(e0, st));
    }
    TWG_CUDA(c, launch_rb_tblock(t, c->tmap[0][t], c->tmap[1][t], a, c->B, (c->row_off + lo) & 1, resid, st));
    if (prof) {
        TWG_CUDA(c, cudaEventRecord(e1, st));
        c->prof_launches += 1;
        c->prof_cells += (int64_t)nscen * c->W * (hi - lo) * t;
    }
    c->launches += 1;
    return TWG_OK;
}

// `to` waits for everything enqueued on `from` so far.
static twg_status join(twg_ctx* c, cudaStream_t from, cudaStream_t to, int slot) {
    if (from == to) return TWG_OK;
    cudaEvent_t e = c->shard.ev[slot];
    TWG_CUDA(c, cudaEventRecord(e, from));
    TWG_CUDA(c, cudaStreamWaitEvent(to, e, 0));
    return TWG_OK;
}

// Buffer holding scenario 0's field after `lp` launches of the current call.
static float* cur_field(twg_ctx* c, int lp) { return c->u[c->cur[0] ^ (lp & 1)]; }

// Ghost-row exchange of a row-slab group: every slab sends its G = 2k owned boundary
// rows to each neighbour and receives the neighbour's into its ghost rows.  NCCL point-to-point
// (one group call per rank) or, for a local group, device copies; enqueued on the comm stream.
static twg_status exchange(const std::vector<twg_ctx*>& g, int lp) {
    twg_ctx* c0 = g[0];
    cudaStream_t cs = c0->shard.comm;
    const int G = c0->ghost;
    if (c0->shard.nccl) {
        twg_ctx* c = c0;
        const size_t cnt = (size_t)G * c->P;
        float* f = cur_field(c, lp);
        const int r = c->shard.rank, n = c->shard.nranks;
        if (n == 1) return TWG_OK;
        return nccl_exchange(c, cnt, r > 0 ? r - 1 : -1, r + 1 < n ? r + 1 : -1, f + (size_t)G * c->P, f,
                             f + (size_t)(c->H - 2 * G) * c->P, f + (size_t)(c->H - G) * c->P, cs);
    }
    for (size_t r = 0; r + 1 < g.size(); ++r) {
        twg_ctx* up = g[r];
        twg_ctx* dn = g[r + 1];
        float* fu = cur_field(up, lp);
        float* fd = cur_field(dn, lp);
        const size_t bytes = (size_t)G * up->P * sizeof(float);
        // up's owned bottom rows -> dn's top ghosts; dn's owned top rows -> up's bottom ghosts
        TWG_CUDA(c0, cudaMemcpyAsync(fd, fu + (size_t)(up->H - 2 * G) * up->P, bytes, cudaMemcpyDeviceToDevice, cs));
        TWG_CUDA(c0, cudaMemcpyAsync(fu + (size_t)(up->H - G) * up->P, fd + (size_t)G * dn->P, bytes,
                                     cudaMemcpyDeviceToDevice, cs));
    }
    return TWG_OK;
}

// Residual max over the slabs of a group (residual bits of the owned rows; floats >= 0 order as
// their bit patterns), enqueued on the comm stream: NCCL all-reduce(max) or a one-block kernel.
static twg_status residual_max(const std::vector<twg_ctx*>& g) {
    twg_ctx* c0 = g[0];
    if (c0->shard.nccl) {
        if (c0->shard.nranks == 1) return TWG_OK;
        return nccl_allreduce_max_u32(c0, c0->d_res_bits, c0->B, c0->shard.comm);
    }
    if (g.size() < 2) return TWG_OK;
    unsigned* ptrs[kMaxLocalSlabs];
    for (size_t r = 0; r < g.size(); ++r) ptrs[r] = g[r]->d_res_bits;
    TWG_CUDA(c0, launch_res_group_max(ptrs, (int)g.size(), c0->B, c0->shard.comm));
    c0->launches += 1;
    return TWG_OK;
}

// Rows a4-a6 for the scenarios whose participation flag is set, on one context or on a row-slab
// group (all slabs of one process: the local group, or this rank's slab of an NCCL group).
// Launches of T sweeps (red-black), single sweeps (Jacobi) or persistent launches (lexicographic),
// then k_check per check interval.  Row slabs run the check interval as exchange
// intervals of at most k sweeps: the j-th launch of an interval writes only the rows still valid
// after it (the ghost region shrinks by 2T rows per launch), the last launch of an interval is split
// into the two boundary bands (comm stream) and the interior (context stream), so that the ghost
// exchange of the boundary rows overlaps the interior tiles; the residual is max-reduced across
// slabs on the device before k_check, so every slab applies the same stop rule without a host hop.
twg_status relax_group(const std::vector<twg_ctx*>& g, const twg_relax_cfg* cfg, const std::vector<int>& part,
                       int* sweeps_done, float* residual) {
    twg_ctx* c0 = g[0];
    if (!cfg) return fail(c0, TWG_E_INVALID_ARG, "null relax cfg");
    const int maxs = cfg->max_sweeps;
    if (maxs < 0 || cfg->check_every < 0) return fail(c0, TWG_E_INVALID_ARG, "negative sweep counts");
    if (cfg->mode < 0 || cfg->mode > 2) return fail(c0, TWG_E_INVALID_ARG, "relax mode must be 0, 1 or 2");
    const bool jacobi = cfg->mode == 1;
    const bool lex = cfg->mode == 2;
    const bool sh = c0->sharded();
    if (lex && c0->ghost > 0) return fail(c0, TWG_E_INVALID_ARG, "lexicographic mode is not available on a row slab");
    if (lex) {
        twg_status ls = ensure_lex(c0);
        if (ls != TWG_OK) return ls;
    }
    const int B = c0->B;
    // sweeps per tile launch: 6 where the launch fills the GPU (issue-bound); small fields
    // (<= 2^20 cells in all: the launch's few warps are latency-bound) take 5 -- C2 512^2, 100 sweeps:
    // 119.8 us at T = 5 vs 129.0 at 6, 122.1 at 4 (and 100 = 20 x 5 needs no remainder launch)
    int T = cfg->temporal_depth > 0 ? std::min(cfg->temporal_depth, kMaxT)
                                    : (!sh && (int64_t)c0->W * c0->H * B <= (int64_t)1 << 20 ? 5 : 6);
    const float tol = cfg->tol;
    int check = (tol > 0.0f && cfg->check_every > 0) ? cfg->check_every : std::max(maxs, 1);
    const int sync_every = cfg->sync_every > 0 ? cfg->sync_every : 64;
    const int kx = sh ? c0->shard.k : std::numeric_limits<int>::max();  // sweeps between exchanges
    cudaStream_t ms = c0->stream, cs = sh ? c0->shard.comm : c0->stream;
    // control arrays [done | cur | sweeps | where | res bits | res]: when the buffer indices or the
    // participation changed since the last call, one copy of the whole block; otherwise a kernel
    // resets done / sweeps / where / residual, so consecutive relaxations stay a chain of kernels
    // (PDL included)
    int nscen = 0;
    for (int b = 0; b < B; ++b) nscen += part[b] ? 1 : 0;
    for (twg_ctx* c : g) {
        bool all = true;
        for (int b = 0; b < B; ++b) all = all && part[b];
        bool same = (int)c->cur_cache.size() == B && (int)c->part_cache.size() == B;
        for (int b = 0; same && b < B; ++b) same = c->cur_cache[b] == c->cur[b] && c->part_cache[b] == (part[b] ? 1 : 0);
        if (!same || !all) {
            int* hs = nullptr;
            TWG_CUDA(c, stage_alloc(c, 6 * B * sizeof(int), reinterpret_cast<void**>(&hs)));
            c->cur_cache.assign(B, 0);
            c->part_cache.assign(B, 0);
            for (int b = 0; b < B; ++b) {
                hs[b] = part[b] ? 0 : 1;
                hs[B + b] = c->cur_cache[b] = c->cur[b];
                c->part_cache[b] = part[b] ? 1 : 0;
                hs[2 * B + b] = 0;
                hs[3 * B + b] = -1;
                hs[4 * B + b] = 0;
                hs[5 * B + b] = 0;  // +0.0f
            }
            TWG_CUDA(c, cudaMemcpyAsync(c->d_ctl, hs, 6 * B * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        } else {
            TWG_CUDA(c, launch_relax_init(c->d_done, c->d_sweeps, c->d_where, c->d_res_bits, c->d_res, B, c->stream));
            c->launches += 1;
        }
    }
    if (lex)
        TWG_CUDA(c0, cudaMemsetAsync(c0->d_lex_tdone, 0, (size_t)B * c0->lex_tx * c0->lex_ty * sizeof(int), ms));
    if (sh) {
        // ghost rows beyond the global grid (top of slab 0, bottom of the last slab) are never
        // exchanged and, with the shrinking launch ranges, never rewritten: keep them obstacle (+0.0,
        // C4) in both ping-pong buffers, since an interval with an odd number of launches leaves
        // the field in the other buffer
        for (twg_ctx* c : g) {
            const size_t bytes = (size_t)c->ghost * c->P * sizeof(float);
            for (int q = 0; q < 2; ++q) {
                if (c->shard.r0 == 0) TWG_CUDA(c, cudaMemsetAsync(c->u[q], 0, bytes, ms));
                if (c->shard.r1 == c->shard.H_global)
                    TWG_CUDA(c, cudaMemsetAsync(c->u[q] + (size_t)(c->H - c->ghost) * c->P, 0, bytes, ms));
            }
        }
    }

    int lp = 0;  // launches so far (parity)
    bool maxs_done_small = false;
    static const bool no_small = [] { const char* e = std::getenv("TWG_NO_SMALL"); return e && e[0] == '1'; }();
    // (an explicit temporal_depth / rows_per_warp asks for the tile kernel)
    if (maxs > 0 && !sh && !jacobi && !lex && !no_small && cfg->temporal_depth == 0 && cfg->rows_per_warp == 0 &&
        small_grid(c0->W, c0->H)) {
        // one CTA per scenario solves the whole relaxation in shared memory (k_rb_small), in place
        RelaxArgs a;
        std::memset(&a, 0, sizeof(a));
        a.u0 = c0->u[0];
        a.u1 = c0->u[1];
        a.cur = c0->d_cur;
        a.P = c0->P;
        a.sstride = c0->sstride;
        a.W = c0->W;
        a.H = c0->H;
        a.done = c0->d_done;
        a.res_r0 = c0->ghost;
        a.res_r1 = c0->H - c0->ghost;
        TWG_CUDA(c0, launch_rb_small(a, B, maxs, check, tol, c0->row_off & 1, c0->d_sweeps, c0->d_res, ms));
        c0->launches += 1;
        maxs_done_small = true;
    }
    if (maxs > 0 && !maxs_done_small) {
        int done_sw = 0, nchunk = 0;
        int lex_base = 0;  // sweeps finished by earlier lexicographic launches of this call
        while (done_sw < maxs) {
            const int chunk = std::min(check, maxs - done_sw);
            for (int in_chunk = 0; in_chunk < chunk;) {
                const int n = std::min(kx, chunk - in_chunk);  // one exchange interval
                const bool resid_iv = in_chunk + n == chunk;    // the chunk's last sweep is in this interval
                // launches of T sweeps, then the remainder; the last launch accumulates the residual
                std::vector<int> plan;
                if (jacobi) {
                    plan.assign(n, 1);
                } else if (lex) {
                    for (int q = 0; q < n / kLexMaxSweeps; ++q) plan.push_back(kLexMaxSweeps);  // persistent launches
                    if (n % kLexMaxSweeps) plan.push_back(n % kLexMaxSweeps);
                } else {
                    for (int q = 0; q < n / T; ++q) plan.push_back(T);
                    if (n % T) plan.push_back(n % T);
                }
                int s = 0;  // sweeps of this interval done after the launch
                // the last launch of the interval is split when every slab is thick enough (the two
                // boundary bands [lo, 2G) and [H - 2G, hi) and a non-empty interior)
                bool split = sh && !jacobi && !lex;
                for (twg_ctx* c : g) split = split && c->ghost > 0 && c->H - 2 * n - 2 * n >= 4 * c->ghost + 2;
                bool split_done = false;
                for (size_t q = 0; q < plan.size(); ++q) {
                    const int t = plan[q];
                    s += t;
                    const bool lastl = q + 1 == plan.size();
                    const bool resid = resid_iv && lastl;
                    if (lex) {
                        int2* tl = lex_tasks(c0, t);
                        if (!tl) return fail(c0, TWG_E_NO_MEMORY, "lexicographic task list");
                        LexArgs la;
                        la.u0 = c0->u[0];
                        la.u1 = c0->u[1];
                        la.cur = c0->d_cur;
                        la.P = c0->P;
                        la.sstride = c0->sstride;
                        la.W = c0->W;
                        la.H = c0->H;
                        la.B = B;
                        la.TX = c0->lex_tx;
                        la.TY = c0->lex_ty;
                        la.ntiles = c0->lex_tx * c0->lex_ty;
                        la.tasks = tl;
                        la.ntasks = t * c0->lex_tx * c0->lex_ty;
                        la.sweeps = t;
                        la.base = lex_base;
                        lex_base += t;
                        la.tdone = c0->d_lex_tdone;
                        la.task = c0->d_lex_task;
                        la.done = c0->d_done;
                        la.res = resid ? c0->d_res_bits : nullptr;  // the chunk's last sweep only
                        la.res_r0 = c0->ghost;
                        la.res_r1 = c0->H - c0->ghost;
                        TWG_CUDA(c0, cudaMemsetAsync(c0->d_lex_task, 0, sizeof(unsigned), ms));
                        TWG_CUDA(c0, launch_lex(la, c0->n_sm, ms));
                        c0->launches += 1;
                        continue;  // the lexicographic sweep is in place (no parity change)
                    }
                    for (twg_ctx* c : g) {
                        if (jacobi) {
                            RelaxArgs a;
                            std::memset(&a, 0, sizeof(a));
                            a.u0 = c->u[0];
                            a.u1 = c->u[1];
                            a.cur = c->d_cur;
                            a.P = c->P;
                            a.sstride = c->sstride;
                            a.W = c->W;
                            a.H = c->H;
                            a.done = c->d_done;
                            a.res = c->d_res_bits;
                            a.res_r0 = c->ghost;
                            a.res_r1 = c->H - c->ghost;
                            a.lp = lp & 1;
                            TWG_CUDA(c, launch_jacobi(a, B, resid, c->stream));
                            c->launches += 1;
                            continue;
                        }
                        // rows valid after s sweeps of the interval: all but 2s at each edge of a slab
                        const int lo = sh ? 2 * s : 0, hi = sh ? c->H - 2 * s : c->H;
                        const int G = c->ghost;
                        if (split && lastl) {
                            // boundary bands first on the comm stream (the exchange reads them), the
                            // interior on the context stream
                            if (c == g[0]) {
                                twg_status js = join(c0, ms, cs, 0);
                                if (js != TWG_OK) return js;
                            }
                            twg_status r1 = launch_rb_range(c, cfg, t, lp, lo, 2 * G, resid, nscen, cs);
                            if (r1 != TWG_OK) return r1;
                            r1 = launch_rb_range(c, cfg, t, lp, c->H - 2 * G, hi, resid, nscen, cs);
                            if (r1 != TWG_OK) return r1;
                            r1 = launch_rb_range(c, cfg, t, lp, 2 * G, c->H - 2 * G, resid, nscen, ms);
                            if (r1 != TWG_OK) return r1;
                            split_done = true;
                        } else {
                            twg_status r1 = launch_rb_range(c, cfg, t, lp, lo, hi, resid, nscen, ms);
                            if (r1 != TWG_OK) return r1;
                        }
                    }
                    ++lp;
                }
                if (sh) {
                    // ghost exchange after every interval (the last one too: ghosts then hold the
                    // neighbours' final rows for the slab walk); the boundary rows were written on
                    // the comm stream when the last launch was split, otherwise wait for the launch
                    if (!split_done) {
                        twg_status js = join(c0, ms, cs, 0);
                        if (js != TWG_OK) return js;
                    }
                    twg_status xs = exchange(g, lp);
                    if (xs != TWG_OK) return xs;
                    if (resid_iv) {
                        twg_status js = join(c0, ms, cs, 1);  // the interior's residual
                        if (js != TWG_OK) return js;
                        twg_status rs = residual_max(g);
                        if (rs != TWG_OK) return rs;
                    }
                    twg_status js = join(c0, cs, ms, 2);
                    if (js != TWG_OK) return js;
                }
                in_chunk += n;
            }
            for (twg_ctx* c : g) {
                TWG_CUDA(c, launch_check(B, c->d_done, c->d_sweeps, c->d_res_bits, c->d_res, c->d_where, chunk, check,
                                         maxs, tol, c->d_cur, lp & 1, c->stream));
                c->launches += 1;
            }
            done_sw += chunk;
            ++nchunk;
            if (tol > 0.0f && done_sw < maxs && nchunk % sync_every == 0) {
                // every slab took the same decision (reduced residual): reading slab 0 suffices
                int* hd = nullptr;
                TWG_CUDA(c0, stage_alloc(c0, B * sizeof(int), reinterpret_cast<void**>(&hd)));
                TWG_CUDA(c0, cudaMemcpyAsync(hd, c0->d_done, B * sizeof(int), cudaMemcpyDeviceToHost, ms));
                TWG_CUDA(c0, cudaStreamSynchronize(ms));
                bool all = true;
                for (int b = 0; b < B; ++b) all = all && hd[b];
                if (all) break;
            }
        }
        if (tol > 0.0f) {  // only an early stop can leave a field in the other buffer
            for (twg_ctx* c : g) {
                TWG_CUDA(c, launch_fixup(c->u[0], c->u[1], c->sstride, B, c->d_where, c->d_cur, lp & 1, c->stream));
                c->launches += 1;
            }
            if (sh) {  // the fixup moved whole fields: refresh the ghosts from the final owned rows
                twg_status js = join(c0, ms, cs, 0);
                if (js != TWG_OK) return js;
                twg_status xs = exchange(g, lp);
                if (xs != TWG_OK) return xs;
                js = join(c0, cs, ms, 2);
                if (js != TWG_OK) return js;
            }
        }
        for (twg_ctx* c : g)
            for (int b = 0; b < B; ++b)
                if (part[b]) c->cur[b] ^= (lp & 1);
    }
    if (sweeps_done || residual) {
        int* hsw = nullptr;  // [sweeps | where | res bits | res] in one copy
        TWG_CUDA(c0, stage_alloc(c0, 4 * B * sizeof(int), reinterpret_cast<void**>(&hsw)));
        float* hr = reinterpret_cast<float*>(hsw + 3 * B);
        TWG_CUDA(c0, cudaMemcpyAsync(hsw, c0->d_sweeps, 4 * B * sizeof(int), cudaMemcpyDeviceToHost, ms));
        TWG_CUDA(c0, cudaStreamSynchronize(ms));
        for (int b = 0; b < B; ++b) {
            if (sweeps_done) sweeps_done[b] = hsw[b];
            if (residual) residual[b] = hr[b];
        }
    }
    return TWG_OK;
}

twg_status relax(twg_ctx* c, const twg_relax_cfg* cfg, const std::vector<int>& part, int* sweeps_done,
                 float* residual) {
    if (!c->shard.peers.empty()) return relax_group(c->shard.peers, cfg, part, sweeps_done, residual);
    return relax_group({c}, cfg, part, sweeps_done, residual);
}

// Rows a7-a9 for a list of scenarios (path kernels only; results stay on device).
twg_status path(twg_ctx* c, const std::vector<int>& bs, const twg_band_cfg* cfg) {
    if (!cfg) return fail(c, TWG_E_INVALID_ARG, "null band cfg");
    if (cfg->max_len < 1 || cfg->max_smooth < 1 || cfg->iterations < 0 || cfg->iterations > 6000)
        return fail(c, TWG_E_INVALID_ARG, "band cfg: max_len, max_smooth >= 1, 0 <= iterations <= 6000");
    twg_status st = ensure_path_cap(c, cfg->max_len, cfg->max_smooth);
    if (st != TWG_OK) return st;
    const int ns = (int)bs.size();
    st = ensure_params(c, ns);
    if (st != TWG_OK) return st;
    std::vector<ScenParams> ps(ns);
    for (int k = 0; k < ns; ++k) {
        const twg_ctx::Scen& sc = c->scen[bs[k]];
        if (!sc.encoded) return fail(c, TWG_E_INVALID_ARG, "extract_path before set_obstacles");
        std::memset(&ps[k], 0, sizeof(ScenParams));
        ps[k].b = bs[k];
        ps[k].gx = sc.gx;
        ps[k].gy = sc.gy;
        ps[k].rcx = sc.rcx;
        ps[k].rcy = sc.rcy;
        ps[k].cur = c->cur[bs[k]];
    }
    void* hp = nullptr;
    TWG_CUDA(c, stage_alloc(c, ns * sizeof(ScenParams), &hp));
    std::memcpy(hp, ps.data(), ns * sizeof(ScenParams));
    TWG_CUDA(c, cudaMemcpyAsync(c->d_params, hp, ns * sizeof(ScenParams), cudaMemcpyHostToDevice, c->stream));
    PathArgs p;
    p.u0 = c->u[0];
    p.u1 = c->u[1];
    p.P = c->P;
    p.sstride = c->sstride;
    p.W = c->W;
    p.H = c->H;
    p.params = c->d_params;
    p.nscen = ns;
    p.max_len = cfg->max_len;
    p.max_smooth = cfg->max_smooth;
    p.iters = cfg->iterations;
    p.step = cfg->step;
    p.kt = cfg->k_t;
    p.cells = c->d_cells;
    p.wp = c->d_wp;
    p.smooth = c->d_smooth;
    p.len_cap = c->path_len_cap;
    p.smooth_cap = c->smooth_cap;
    p.meta = c->d_meta;
    p.dir = c->d_dir;
    p.istride = c->sstride;
    p.dir_map = c->dir_map;
    // speculative segment walkers from markers on the previous path (k_index_dir); TWG_NO_SPEC=1
    // runs the single walker only (same results)
    static const bool no_spec = [] { const char* e = std::getenv("TWG_NO_SPEC"); return e && e[0] == '1'; }();
    p.spec = c->d_spec;
    p.seg = c->d_seg;
    p.seg_cells = c->d_seg_cells;
    p.spec_on = (!no_spec && c->d_seg_cells) ? 1 : 0;
    int nl = 0;
    TWG_CUDA(c, launch_path(p, &nl, c->stream));
    c->launches += nl;
    return TWG_OK;
}

// Row f1 tick for the requests rq (det_off relative to `det`, a device array of (x, y) pairs).
twg_status track_core(twg_ctx* c, std::vector<TrkReq> rq, const double2* det, const twg_warp_cfg* wc,
                      const twg_tracker_cfg* cfg, std::vector<int>& n_out) {
    twg_status st = TWG_OK;
    const int nreq = (int)rq.size();
    n_out.clear();
    if (nreq == 0) return TWG_OK;
    int max_n = 0, max_m = 0, need_cap = 1;
    for (const TrkReq& r : rq) {
        max_n = std::max(max_n, r.n);
        max_m = std::max(max_m, r.m);
        need_cap = std::max(need_cap, r.n + r.m);
    }
    st = ensure_track_cap(c, need_cap);
    if (st != TWG_OK) return st;
    for (int k = 0; k < nreq; ++k)
        rq[k].limit = cfg->max_tracks > 0 ? std::min(cfg->max_tracks, c->track_cap) : c->track_cap;
    // scratch: [B][cap] tables, [nreq][mcap] flags, [nreq][pcap] pairs, control words, requests, detections
    if (c->trk_scratch_cap < c->track_cap) {
        for (void* p : {(void*)c->d_trk_pred, (void*)c->d_trk_misn, (void*)c->d_trk_match})
            if (p) cudaFree(p);
        c->d_trk_pred = nullptr;
        c->d_trk_misn = c->d_trk_match = nullptr;
        TWG_CUDA(c, dev_alloc(&c->d_trk_pred, (size_t)c->B * c->track_cap));
        TWG_CUDA(c, dev_alloc(&c->d_trk_misn, (size_t)c->B * c->track_cap));
        TWG_CUDA(c, dev_alloc(&c->d_trk_match, (size_t)c->B * c->track_cap));
        c->trk_scratch_cap = c->track_cap;
    }
    int pcap = 4096;
    while (pcap < 4 * (max_n + max_m)) pcap <<= 1;
    pcap = std::max(pcap, c->trk_pcap);
    const int mcap = std::max(max_m, 1);
    auto alloc_req_scratch = [&](int pc) -> twg_status {
        if (c->trk_nreq_cap < nreq || c->trk_mcap < mcap) {
            if (c->d_trk_used) cudaFree(c->d_trk_used);
            c->d_trk_used = nullptr;
            TWG_CUDA(c, dev_alloc(&c->d_trk_used, (size_t)std::max(nreq, c->trk_nreq_cap) * std::max(mcap, c->trk_mcap)));
            c->trk_mcap = std::max(mcap, c->trk_mcap);
        }
        if (c->trk_nreq_cap < nreq || c->trk_pcap < pc) {
            if (c->d_trk_pairs) cudaFree(c->d_trk_pairs);
            c->d_trk_pairs = nullptr;
            TWG_CUDA(c, dev_alloc(&c->d_trk_pairs, (size_t)std::max(nreq, c->trk_nreq_cap) * std::max(pc, c->trk_pcap)));
            c->trk_pcap = std::max(pc, c->trk_pcap);
        }
        if (c->trk_nreq_cap < nreq) {
            if (c->d_trk_ctl) cudaFree(c->d_trk_ctl);
            if (c->d_trk_req) cudaFree(c->d_trk_req);
            c->d_trk_ctl = nullptr;
            c->d_trk_req = nullptr;
            TWG_CUDA(c, dev_alloc(&c->d_trk_ctl, (size_t)3 * nreq));
            TWG_CUDA(c, dev_alloc(&c->d_trk_req, (size_t)nreq));
            c->trk_nreq_cap = nreq;
        }
        return TWG_OK;
    };
    st = alloc_req_scratch(pcap);
    if (st != TWG_OK) return st;
    TrackArgs t;
    t.trk = c->d_tracks;
    t.missed = c->d_missed;
    t.pred = c->d_trk_pred;
    t.mis_new = c->d_trk_misn;
    t.match = c->d_trk_match;
    t.det = det;
    t.cap = c->track_cap;
    t.mcap = c->trk_mcap;
    t.prune_after = cfg->prune_after;
    std::memcpy(t.Q, wc->Q, sizeof(t.Q));
    t.dt = wc->dt;
    t.r2 = cfg->sigma_z * cfg->sigma_z;
    t.gate2 = cfg->gate * cfg->gate;
    t.var_pos = cfg->spawn_var_pos;
    t.var_vel = cfg->spawn_var_vel;
    std::vector<int> result_n(nreq, 0);
    int worst = 0;
    std::vector<TrkReq> todo = rq;
    std::vector<int> todo_idx(nreq);
    for (int k = 0; k < nreq; ++k) todo_idx[k] = k;
    for (int attempt = 0; !todo.empty(); ++attempt) {
        const int nr = (int)todo.size();
        int mn = 0, mm = 0;
        for (const TrkReq& r : todo) {
            mn = std::max(mn, r.n);
            mm = std::max(mm, r.m);
        }
        void* hq = nullptr;
        TWG_CUDA(c, stage_alloc(c, nr * sizeof(TrkReq), &hq));
        std::memcpy(hq, todo.data(), nr * sizeof(TrkReq));
        TWG_CUDA(c, cudaMemcpyAsync(c->d_trk_req, hq, nr * sizeof(TrkReq), cudaMemcpyHostToDevice, c->stream));
        TWG_CUDA(c, cudaMemsetAsync(c->d_trk_ctl, 0, 3 * nr * sizeof(int), c->stream));
        t.req = c->d_trk_req;
        t.used = c->d_trk_used;
        t.pairs = c->d_trk_pairs;
        t.pcap = c->trk_pcap;
        t.pcount = c->d_trk_ctl;
        t.flags = c->d_trk_ctl + nr;
        t.n_out = c->d_trk_ctl + 2 * nr;
        int nl = 0;
        TWG_CUDA(c, launch_track_step(t, nr, mn, mm, &nl, c->stream));
        c->launches += nl;
        int* hc = nullptr;
        TWG_CUDA(c, stage_alloc(c, 3 * nr * sizeof(int), reinterpret_cast<void**>(&hc)));
        TWG_CUDA(c, cudaMemcpyAsync(hc, c->d_trk_ctl, 3 * nr * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        TWG_CUDA(c, cudaStreamSynchronize(c->stream));
        std::vector<TrkReq> again;
        std::vector<int> again_idx;
        int need = 0;
        for (int q = 0; q < nr; ++q) {
            const int fl = hc[nr + q];
            if (fl & kTrkOverflow) {  // more gated pairs than the list holds: grow and redo this scenario
                again.push_back(todo[q]);
                again_idx.push_back(todo_idx[q]);
                need = std::max(need, hc[q]);
                continue;
            }
            result_n[todo_idx[q]] = hc[2 * nr + q];
            c->scen[todo[q].b].trk_n = hc[2 * nr + q];
            if (fl & kTrkSingular) worst = std::max(worst, (int)TWG_W_SINGULAR_INNOVATION);
            if (fl & kTrkTruncated) worst = std::max(worst, (int)TWG_W_TRUNCATED);
        }
        if (!again.empty()) {
            if (attempt > 40) return fail(c, TWG_E_NO_MEMORY, "tracker pair list cannot grow");
            int pc = c->trk_pcap;
            while (pc < need) pc <<= 1;
            st = alloc_req_scratch(pc);
            if (st != TWG_OK) return st;
        }
        todo.swap(again);
        todo_idx.swap(again_idx);
    }
    n_out.assign(result_n.begin(), result_n.end());
    return (twg_status)worst;
}


}  // namespace host
}  // namespace twg
