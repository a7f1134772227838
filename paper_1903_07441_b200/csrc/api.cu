// api.cu -- the core entry points of include/twg.h (context, rows a1-a9, field access, accounting).
// Helpers and the a1-a9 orchestration are in host_core.cu; the 8(f) rows in api_track.cu (f1),
// api_sim.cu (f2) and api_extra.cu (f3, slab walk).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "api_host.cuh"

using namespace twg;
using namespace twg::host;


// =====================================================================================
// Allocate and initialise a context for the local grid `d` (unsharded, or one slab).
static twg_status create_local(const twg_grid_desc* d, int32_t device, void* stream, twg_ctx** out) {
    *out = nullptr;
    if (d->width <= 0 || d->height <= 0 || d->batch <= 0 || !(d->cell_size > 0.0))
        return fail(nullptr, TWG_E_INVALID_ARG, "width, height, batch > 0 and cell_size > 0 required");
    if (d->batch > 65535 || d->width >= (1 << 24) || d->height >= (1 << 24))
        return fail(nullptr, TWG_E_INVALID_ARG, "batch <= 65535 (one grid dimension per scenario) and sides < 2^24");
    if (d->ghost_rows < 0 || 2 * d->ghost_rows >= d->height)
        return fail(nullptr, TWG_E_INVALID_ARG, "0 <= ghost_rows < height / 2 required");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(nullptr, TWG_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    twg_ctx* c = new twg_ctx();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    if (cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || c->n_sm <= 0)
        c->n_sm = 148;
    c->W = d->width;
    c->H = d->height;
    c->B = d->batch;
    c->row_off = d->row_offset;
    c->ghost = d->ghost_rows;
    c->cs = d->cell_size;
    c->ox = d->origin_x;
    c->oy = d->origin_y;
    c->P = ((int64_t)c->W + 31) / 32 * 32;
    c->sstride = c->P * c->H;
    c->cur.assign(c->B, 0);
    c->scen.assign(c->B, twg_ctx::Scen());
    const size_t B = c->B, cells = (size_t)c->sstride * B;
    auto bail = [&](twg_status st, const std::string& m) {
        g_create_err = m;
        twg_destroy(c);
        return st;
    };
#define CK(expr)                                                                                      \
    do {                                                                                              \
        cudaError_t e_ = (expr);                                                                      \
        if (e_ != cudaSuccess)                                                                        \
            return bail(e_ == cudaErrorMemoryAllocation ? TWG_E_NO_MEMORY : TWG_E_CUDA,               \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                          \
    } while (0)
    CK(dev_alloc(&c->u[0], cells));
    CK(dev_alloc(&c->u[1], cells));
    CK(dev_alloc(&c->mask, B * c->H * c->W));
    CK(dev_alloc(&c->d_ctl, 7 * B));
    CK(cudaMemset(c->d_ctl, 0, 7 * B * sizeof(int)));
    c->d_done = c->d_ctl;
    c->d_cur = c->d_ctl + B;
    c->d_sweeps = c->d_ctl + 2 * B;
    c->d_where = c->d_ctl + 3 * B;
    c->d_res_bits = reinterpret_cast<unsigned*>(c->d_ctl + 4 * B);
    c->d_res = reinterpret_cast<float*>(c->d_ctl + 5 * B);
    c->d_flags = c->d_ctl + 6 * B;
    CK(dev_alloc(&c->d_fixbox, 2 * B));
    {
        std::vector<int4> empty(2 * B, make_int4(1, 0, 1, 0));  // no positive fixed cell yet
        CK(cudaMemcpy(c->d_fixbox, empty.data(), 2 * B * sizeof(int4), cudaMemcpyHostToDevice));
    }
    CK(dev_alloc(&c->d_meta, B));
    CK(dev_alloc(&c->d_dir, cells));
    CK(cudaMemsetAsync(c->mask, 0, B * c->H * c->W, c->stream));
    CK(cudaMemsetAsync(c->d_meta, 0, B * sizeof(PathMeta), c->stream));
    static unsigned long long preloaded = 0;  // eager module loading, once per device
    if (first_on_device(preloaded)) {
        preload_relax_kernels();
        preload_stamp_kernels();
        preload_path_kernels();
        preload_track_kernels();
        preload_sim_kernels();
    }
    CK(launch_init_field(c->u[0], c->P, c->sstride, c->W, c->H, c->B, c->stream));
    CK(launch_init_field(c->u[1], c->P, c->sstride, c->W, c->H, c->B, c->stream));
    c->launches += 2;
    c->hmask.assign(B * c->H * c->W, 0);
    for (int t = 1; t <= kMaxT; ++t)
        if (!make_tmap(&c->tmap[0][t], c->u[0], c->W, c->H, c->B, c->P, 2 * t + 2) ||
            !make_tmap(&c->tmap[1][t], c->u[1], c->W, c->H, c->B, c->P, 2 * t + 2))
            return bail(TWG_E_CUDA, "cuTensorMapEncodeTiled failed (driver entry point unavailable or bad layout)");
    if (!make_dir_map(&c->dir_map, c->d_dir, c->H, c->B, c->P))
        return bail(TWG_E_CUDA, "cuTensorMapEncodeTiled failed for the index matrix");
    CK(cudaStreamSynchronize(c->stream));
#undef CK
    *out = c;
    return TWG_OK;
}

// Comm stream (highest priority) and join events of a row-slab context or local group.
struct SlabStreams {
    cudaStream_t comm = nullptr;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    ~SlabStreams() {
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (comm) cudaStreamDestroy(comm);
    }
};

static twg_status make_streams(std::shared_ptr<void>* out) {
    auto s = std::make_shared<SlabStreams>();
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaError_t e = cudaStreamCreateWithPriority(&s->comm, cudaStreamNonBlocking, hi);
    for (int k = 0; k < 3 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&s->ev[k], cudaEventDisableTiming);
    if (e != cudaSuccess) return fail(nullptr, TWG_E_CUDA, std::string("slab streams: ") + cudaGetErrorString(e));
    *out = s;
    return TWG_OK;
}

static void attach_streams(twg_ctx* c, const std::shared_ptr<void>& s) {
    const SlabStreams* ss = static_cast<const SlabStreams*>(s.get());
    c->shard.streams = s;
    c->shard.comm = ss->comm;
    for (int k = 0; k < 3; ++k) c->shard.ev[k] = ss->ev[k];
}

// Slab `rank` of `nranks` of the global grid d: owned global rows [r0, r1) (near-equal
// contiguous split) plus G = 2k ghost rows per side, local row 0 = global row r0 - G.
static twg_status create_slab(const twg_grid_desc* d, int rank, int nranks, int32_t device, void* stream,
                              twg_ctx** out) {
    const int k = d->exchange_every;
    if (k < 1) return fail(nullptr, TWG_E_INVALID_ARG, "a row-slab context needs exchange_every >= 1");
    if (d->batch != 1 || d->ghost_rows != 0 || d->row_offset != 0)
        return fail(nullptr, TWG_E_INVALID_ARG, "row slabs: batch 1, ghost_rows 0 and row_offset 0 in the global desc");
    const int G = 2 * k;
    const int base = d->height / nranks, extra = d->height % nranks;
    const int r0 = rank * base + std::min(rank, extra);
    const int r1 = r0 + base + (rank < extra ? 1 : 0);
    if (r1 - r0 < G) return fail(nullptr, TWG_E_INVALID_ARG, "slab thinner than 2 exchange_every rows");
    twg_grid_desc l = *d;
    l.height = r1 - r0 + 2 * G;
    l.row_offset = r0 - G;
    l.ghost_rows = G;
    l.origin_y = d->origin_y + (double)(r0 - G) * d->cell_size;
    twg_status st = create_local(&l, device, stream, out);
    if (st != TWG_OK) return st;
    twg_ctx* c = *out;
    c->shard.nranks = nranks;
    c->shard.rank = rank;
    c->shard.k = k;
    c->shard.H_global = d->height;
    c->shard.r0 = r0;
    c->shard.r1 = r1;
    return TWG_OK;
}

TWG_API twg_status twg_create(const twg_grid_desc* d, int32_t device, void* stream, void* nccl_comm, twg_ctx** out) {
    TWG_NVTX("twg_create");
    if (!d || !out) return fail(nullptr, TWG_E_INVALID_ARG, "null argument");
    *out = nullptr;
    if (!nccl_comm) return create_local(d, device, stream, out);
    int rank = 0, nranks = 1;
    twg_status st = nccl_comm_rank(nullptr, nccl_comm, &rank, &nranks);
    if (st != TWG_OK) return st;
    std::shared_ptr<void> ss;
    st = make_streams(&ss);
    if (st != TWG_OK) return st;
    st = create_slab(d, rank, nranks, device, stream, out);
    if (st != TWG_OK) return st;
    (*out)->shard.nccl = nccl_comm;
    attach_streams(*out, ss);
    return TWG_OK;
}

TWG_API twg_status twg_create_group(const twg_grid_desc* d, int32_t nslabs, int32_t device, void* stream,
                                    twg_ctx** out) {
    TWG_NVTX("twg_create_group");
    if (!d || !out || nslabs < 1 || nslabs > kMaxLocalSlabs)
        return fail(nullptr, TWG_E_INVALID_ARG, "null argument or nslabs outside 1..16");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(nullptr, TWG_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    std::shared_ptr<void> ss;
    twg_status st = make_streams(&ss);
    if (st != TWG_OK) return st;
    std::vector<twg_ctx*> g(nslabs, nullptr);
    for (int r = 0; r < nslabs; ++r) {
        st = create_slab(d, r, nslabs, device, stream, &g[r]);
        if (st != TWG_OK) {
            for (twg_ctx* c : g) twg_destroy(c);
            return st;
        }
        attach_streams(g[r], ss);
    }
    for (int r = 0; r < nslabs; ++r) {
        g[r]->shard.peers = g;
        out[r] = g[r];
    }
    return TWG_OK;
}

TWG_API twg_status twg_slab_info(const twg_ctx* c, int32_t* out8) {
    TWG_NVTX("twg_slab_info");
    if (!c || !out8) return TWG_E_INVALID_ARG;
    const bool sh = c->sharded();
    out8[0] = sh ? c->shard.rank : 0;
    out8[1] = sh ? c->shard.nranks : 1;
    out8[2] = sh ? c->shard.r0 : c->row_off + c->ghost;
    out8[3] = sh ? c->shard.r1 : c->row_off + c->H - c->ghost;
    out8[4] = c->row_off;
    out8[5] = c->ghost;
    out8[6] = sh ? c->shard.k : 0;
    out8[7] = c->H;
    return TWG_OK;
}

TWG_API twg_status twg_destroy(twg_ctx* c) {
    TWG_NVTX("twg_destroy");
    if (!c) return TWG_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    // a slab leaving its local group breaks the group: the other slabs forget their peers
    for (twg_ctx* p : c->shard.peers)
        if (p != c) p->shard.peers.clear();
    void* ptrs[] = {c->u[0],     c->u[1],      c->mask,    c->d_ctl,   c->d_meta,   c->d_tracks,   c->d_t,
                    c->d_j,      c->d_pred,    c->d_boxes, c->d_param_block, c->d_track_off, c->d_cells, c->d_wp,
                    c->d_smooth, c->d_track_tmp, c->d_dir, c->d_fixbox, c->d_missed, c->d_trk_pred, c->d_trk_misn,
                    c->d_trk_match, c->d_trk_used, c->d_trk_pairs, c->d_trk_ctl, c->d_trk_req, c->d_trk_det,
                    c->d_sim_rob, c->d_sim_int, c->d_sim_goal, c->d_sim_nobs, c->d_sim_obs, c->d_sim_obs_old,
                    c->d_sim_speed, c->d_sim_det, c->d_sim_hist, c->d_lex_tdone, c->d_lex_task, c->d_spec,
                    c->d_seg, c->d_seg_cells};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (auto& e : c->lex_lists) cudaFree(e.second);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    delete c;
    return TWG_OK;
}

TWG_API twg_status twg_set_static(twg_ctx* c, int32_t b, const uint8_t* occ) {
    TWG_NVTX("twg_set_static");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!occ || b < -1 || b >= c->B) return fail(c, TWG_E_INVALID_ARG, "bad scenario index or null mask");
    const size_t n = (size_t)c->H * c->W;
    const bool dev = is_device_ptr(occ);
    const int b0 = b < 0 ? 0 : b, b1 = b < 0 ? c->B : b + 1;
    if (c->sharded()) {
        // occ is the global H_global x W mask: take the local rows, rows outside the grid are walls (C4)
        const size_t W = c->W;
        for (int y = 0; y < c->H; ++y) {
            const int gy = c->row_off + y;
            uint8_t* dst = c->hmask.data() + (size_t)y * W;
            if (gy < 0 || gy >= c->shard.H_global) std::memset(dst, 1, W);
            else if (dev) TWG_CUDA(c, cudaMemcpy(dst, occ + (size_t)gy * W, W, cudaMemcpyDeviceToHost));
            else std::memcpy(dst, occ + (size_t)gy * W, W);
        }
        TWG_CUDA(c, cudaMemcpyAsync(c->mask, c->hmask.data(), n, cudaMemcpyHostToDevice, c->stream));
        c->scen[0].static_dirty = true;
        TWG_CUDA(c, cudaStreamSynchronize(c->stream));
        return TWG_OK;
    }
    for (int q = b0; q < b1; ++q) {
        if (dev) {
            TWG_CUDA(c, cudaMemcpyAsync(c->mask + q * n, occ, n, cudaMemcpyDeviceToDevice, c->stream));
            TWG_CUDA(c, cudaMemcpyAsync(c->hmask.data() + q * n, occ, n, cudaMemcpyDeviceToHost, c->stream));
        } else {
            std::memcpy(c->hmask.data() + q * n, occ, n);
            TWG_CUDA(c, cudaMemcpyAsync(c->mask + q * n, c->hmask.data() + q * n, n, cudaMemcpyHostToDevice, c->stream));
        }
        c->scen[q].static_dirty = true;
    }
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

TWG_API twg_status twg_set_obstacles(twg_ctx* c, int32_t b, const twg_robot* robot, int32_t goal_x, int32_t goal_y,
                                     const twg_track* tracks, int32_t n, const twg_warp_cfg* cfg, int32_t warm) {
    TWG_NVTX("twg_set_obstacles");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!robot || b < 0 || b >= c->B || (n > 0 && !tracks)) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    const bool resident = !tracks && n == TWG_RESIDENT_TRACKS;
    if (resident) n = c->scen[b].trk_n;
    if (c->sharded()) goal_y -= c->row_off;  // global goal row -> local
    EncodeReq r{b, *robot, goal_x, goal_y, n, 0};
    st = encode(c, {r}, tracks, cfg, warm, resident);
    if (st != TWG_OK) return st;
    int* hf = nullptr;
    TWG_CUDA(c, stage_alloc(c, sizeof(int), reinterpret_cast<void**>(&hf)));
    TWG_CUDA(c, cudaMemcpyAsync(hf, c->d_flags + b, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    const int flag = *hf;
    return flag ? TWG_W_GOAL_SWALLOWED : TWG_OK;
}

TWG_API twg_status twg_relax(twg_ctx* c, const twg_relax_cfg* cfg, int32_t* sweeps_done, float* residual) {
    TWG_NVTX("twg_relax");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    std::vector<int> part(c->B, 1);
    return relax(c, cfg, part, sweeps_done, residual);
}

TWG_API twg_status twg_extract_path(twg_ctx* c, int32_t b, const twg_band_cfg* cfg, int32_t* cells_xy,
                                    int32_t* n_cells, float* smooth_xy, int32_t* n_smooth, float* next_xy) {
    TWG_NVTX("twg_extract_path");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (b < 0 || b >= c->B) return fail(c, TWG_E_INVALID_ARG, "bad scenario index");
    if (c->sharded()) {
        if (!cfg || cfg->max_len < 1 || cfg->max_smooth < 1 || cfg->iterations < 0 || cfg->iterations > 6000)
            return fail(c, TWG_E_INVALID_ARG, "band cfg: max_len, max_smooth >= 1, 0 <= iterations <= 6000");
        return sharded_extract_path(c, cfg, cells_xy, n_cells, smooth_xy, n_smooth, next_xy);
    }
    if (c->ghost > 0) return fail(c, TWG_E_INVALID_ARG, "path extraction is not available on a manual row slab");
    st = path(c, {b}, cfg);
    if (st != TWG_OK) return st;
    PathMeta* hm = nullptr;
    TWG_CUDA(c, stage_alloc(c, sizeof(PathMeta), reinterpret_cast<void**>(&hm)));
    TWG_CUDA(c, cudaMemcpyAsync(hm, c->d_meta + b, sizeof(PathMeta), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    const PathMeta m = *hm;
    if (cells_xy && m.n_cells > 0)
        TWG_CUDA(c, cudaMemcpyAsync(cells_xy, c->d_cells + (int64_t)b * c->path_len_cap, m.n_cells * sizeof(int2),
                                    cudaMemcpyDeviceToHost, c->stream));
    const int ns = std::min(m.n_smooth, cfg->max_smooth);
    if (smooth_xy && ns > 0)
        TWG_CUDA(c, cudaMemcpyAsync(smooth_xy, c->d_smooth + (int64_t)b * c->smooth_cap, ns * sizeof(float2),
                                    cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    if (n_cells) *n_cells = m.n_cells;
    if (n_smooth) *n_smooth = m.n_smooth;
    if (next_xy) {
        next_xy[0] = m.next_x;
        next_xy[1] = m.next_y;
    }
    if (m.status != TWG_OK) return fail(c, TWG_E_NO_PATH, "no path: the walk entered an obstacle or exceeded max_len");
    return m.n_smooth > cfg->max_smooth ? TWG_W_TRUNCATED : TWG_OK;
}

TWG_API twg_status twg_plan_step(twg_ctx* c, int32_t b, const twg_robot* robot, const int32_t* goal_xy,
                                 const twg_track* tracks, const int32_t* n_tracks, const twg_warp_cfg* warp,
                                 const twg_relax_cfg* rcfg, const twg_band_cfg* bcfg, twg_plan_result* out,
                                 int32_t* cells_xy, float* smooth_xy) {
    TWG_NVTX("twg_plan_step");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!robot || !goal_xy || !rcfg || !bcfg || !out || b < -1 || b >= c->B)
        return fail(c, TWG_E_INVALID_ARG, "bad argument");
    const bool resident = !tracks && !n_tracks;
    if (!n_tracks && !resident) return fail(c, TWG_E_INVALID_ARG, "null n_tracks");
    if (c->ghost > 0) return fail(c, TWG_E_INVALID_ARG, "twg_plan_step is not available on a row slab");
    std::vector<EncodeReq> reqs;
    std::vector<int> bs;
    int64_t off = 0;
    const int ns = b < 0 ? c->B : 1;
    for (int k = 0; k < ns; ++k) {
        const int bk = b < 0 ? k : b;
        const int nk = resident ? c->scen[bk].trk_n : n_tracks[k];
        EncodeReq r{bk, robot[k], goal_xy[2 * k], goal_xy[2 * k + 1], nk, off};
        off += nk;
        reqs.push_back(r);
        bs.push_back(r.b);
    }
    if (off > 0 && !tracks && !resident) return fail(c, TWG_E_INVALID_ARG, "null tracks");
    {
        TWG_NVTX("twg_plan_step/encode");
        st = encode(c, reqs, tracks, warp, rcfg->warm_start, resident);
    }
    if (st != TWG_OK) return st;
    std::vector<int> part(c->B, 0);
    for (int q : bs) part[q] = 1;
    {
        TWG_NVTX("twg_plan_step/relax");
        st = relax(c, rcfg, part, nullptr, nullptr);
    }
    if (st != TWG_OK) return st;
    {
        TWG_NVTX("twg_plan_step/path");
        st = path(c, bs, bcfg);
    }
    if (st != TWG_OK) return st;
    // D2H: per scenario meta, sweeps, residual, flags (pinned staging), then the paths
    const int B = c->B;
    const size_t mb = B * sizeof(PathMeta);
    char* h = nullptr;
    TWG_CUDA(c, stage_alloc(c, mb + 5 * B * sizeof(int), reinterpret_cast<void**>(&h)));
    PathMeta* hm = reinterpret_cast<PathMeta*>(h);
    int* hsw = reinterpret_cast<int*>(h + mb);  // [sweeps | where | res bits | res | flags] in one copy
    float* hr = reinterpret_cast<float*>(hsw + 3 * B);
    int* hf = hsw + 4 * B;
    TWG_CUDA(c, cudaMemcpyAsync(hm, c->d_meta, mb, cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaMemcpyAsync(hsw, c->d_sweeps, 5 * B * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (b < 0) {  // batch: whole capacity per scenario, one strided copy each
        if (cells_xy)
            TWG_CUDA(c, cudaMemcpy2DAsync(cells_xy, bcfg->max_len * sizeof(int2), c->d_cells,
                                          c->path_len_cap * sizeof(int2), bcfg->max_len * sizeof(int2), B,
                                          cudaMemcpyDeviceToHost, c->stream));
        if (smooth_xy)
            TWG_CUDA(c, cudaMemcpy2DAsync(smooth_xy, bcfg->max_smooth * sizeof(float2), c->d_smooth,
                                          c->smooth_cap * sizeof(float2), bcfg->max_smooth * sizeof(float2), B,
                                          cudaMemcpyDeviceToHost, c->stream));
    }
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    // copy the per-scenario results out of the staging ring now: the path read-back below takes a
    // second staging region, which may wrap over (or reallocate) this one
    const std::vector<PathMeta> vm(hm, hm + B);
    const std::vector<int> vsw(hsw, hsw + B), vf(hf, hf + B);
    const std::vector<float> vr(hr, hr + B);
    if (b >= 0 && (cells_xy || smooth_xy) && vm[b].status == TWG_OK) {
        // one scenario: read back only the cells and points produced, through the pinned staging
        // buffer (the caller's arrays are usually pageable)
        const int nc = std::min(vm[b].n_cells, bcfg->max_len);
        const int nsm = std::min(vm[b].n_smooth, bcfg->max_smooth);
        const size_t bc = cells_xy ? (size_t)nc * sizeof(int2) : 0, bsm = smooth_xy ? (size_t)nsm * sizeof(float2) : 0;
        char* hp = nullptr;
        TWG_CUDA(c, stage_alloc(c, bc + bsm + 16, reinterpret_cast<void**>(&hp)));
        if (bc) TWG_CUDA(c, cudaMemcpyAsync(hp, c->d_cells + (int64_t)b * c->path_len_cap, bc, cudaMemcpyDeviceToHost,
                                            c->stream));
        if (bsm)
            TWG_CUDA(c, cudaMemcpyAsync(hp + bc, c->d_smooth + (int64_t)b * c->smooth_cap, bsm,
                                        cudaMemcpyDeviceToHost, c->stream));
        TWG_CUDA(c, cudaStreamSynchronize(c->stream));
        if (bc) std::memcpy(cells_xy, hp, bc);
        if (bsm) std::memcpy(smooth_xy, hp + bc, bsm);
    }
    twg_status worst = TWG_OK;
    for (int k = 0; k < ns; ++k) {
        const int q = bs[k];
        twg_plan_result& r = out[k];
        r.sweeps = vsw[q];
        r.residual = vr[q];
        r.n_cells = vm[q].n_cells;
        r.n_smooth = vm[q].status == TWG_OK ? vm[q].n_smooth : 0;
        r.next_x = vm[q].next_x;
        r.next_y = vm[q].next_y;
        r.walk_status = vm[q].status;
        twg_status s = TWG_OK;
        if (vm[q].status != TWG_OK) s = TWG_E_NO_PATH;
        else if (vf[q]) s = TWG_W_GOAL_SWALLOWED;
        else if (r.n_smooth > bcfg->max_smooth) s = TWG_W_TRUNCATED;
        r.status = s;
        if (s < 0 ? (worst >= 0 || s < worst) : (worst >= 0 && s > worst)) worst = s;
    }
    if (worst < 0) c->err = "at least one scenario has no path";
    return worst;
}

TWG_API twg_status twg_get_field(twg_ctx* c, int32_t b, float* out, int32_t mode) {
    TWG_NVTX("twg_get_field");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!out || b < 0 || b >= c->B || mode < 0 || mode > 2) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    const float* src = c->u[c->cur[b]] + (int64_t)b * c->sstride;
    const size_t bytes = (size_t)c->W * c->H * sizeof(float);
    if (is_device_ptr(out)) {
        TWG_CUDA(c, launch_convert(src, c->P, c->W, c->H, out, mode, c->stream));
        c->launches += 1;
        TWG_CUDA(c, cudaStreamSynchronize(c->stream));
        return TWG_OK;
    }
    float* tmp = nullptr;
    TWG_CUDA(c, cudaMallocAsync(reinterpret_cast<void**>(&tmp), bytes, c->stream));
    TWG_CUDA(c, launch_convert(src, c->P, c->W, c->H, tmp, mode, c->stream));
    c->launches += 1;
    TWG_CUDA(c, cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaFreeAsync(tmp, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

TWG_API twg_status twg_set_field(twg_ctx* c, int32_t b, const float* raw) {
    TWG_NVTX("twg_set_field");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!raw || b < 0 || b >= c->B) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    float* dst = c->u[c->cur[b]] + (int64_t)b * c->sstride;
    const size_t bytes = (size_t)c->W * c->H * sizeof(float);
    const float* src = raw;
    float* tmp = nullptr;
    if (!is_device_ptr(raw)) {
        TWG_CUDA(c, cudaMallocAsync(reinterpret_cast<void**>(&tmp), bytes, c->stream));
        TWG_CUDA(c, cudaMemcpyAsync(tmp, raw, bytes, cudaMemcpyHostToDevice, c->stream));
        src = tmp;
    }
    int4* hb = nullptr;  // imported-field box: empty, then grown by k_import
    TWG_CUDA(c, stage_alloc(c, sizeof(int4), reinterpret_cast<void**>(&hb)));
    *hb = make_int4(std::numeric_limits<int>::max(), -1, std::numeric_limits<int>::max(), -1);
    TWG_CUDA(c, cudaMemcpyAsync(c->d_fixbox + 2 * b + 1, hb, sizeof(int4), cudaMemcpyHostToDevice, c->stream));
    TWG_CUDA(c, launch_import(src, c->W, c->H, dst, c->P, c->d_fixbox + 2 * b + 1, c->stream));
    c->launches += 1;
    if (tmp) TWG_CUDA(c, cudaFreeAsync(tmp, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

TWG_API twg_status twg_get_warp(twg_ctx* c, int32_t b, int32_t n, int32_t* t, int32_t* j, double* pred) {
    TWG_NVTX("twg_get_warp");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (b < 0 || b >= c->B || n != c->scen[b].n_tracks) return fail(c, TWG_E_INVALID_ARG, "bad scenario or count");
    if (n == 0) return TWG_OK;
    const int64_t o = (int64_t)b * c->track_cap;
    if (t) TWG_CUDA(c, cudaMemcpyAsync(t, c->d_t + o, n * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (j) TWG_CUDA(c, cudaMemcpyAsync(j, c->d_j + o, n * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (pred) TWG_CUDA(c, cudaMemcpyAsync(pred, c->d_pred + 3 * o, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

TWG_API twg_status twg_field_ptr(twg_ctx* c, int32_t b, void** dev_ptr, int64_t* pitch) {
    TWG_NVTX("twg_field_ptr");
    if (!c || b < 0 || b >= c->B) return TWG_E_INVALID_ARG;
    if (dev_ptr) *dev_ptr = c->u[c->cur[b]] + (int64_t)b * c->sstride;
    if (pitch) *pitch = c->P;
    return TWG_OK;
}

TWG_API twg_status twg_debug_walk(twg_ctx* c, int32_t b, int32_t* out4) {
    TWG_NVTX("twg_debug_walk");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!out4 || b < 0 || b >= c->B) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    PathMeta m;
    TWG_CUDA(c, cudaMemcpy(&m, c->d_meta + b, sizeof(PathMeta), cudaMemcpyDeviceToHost));
    out4[0] = m.pad[0];
    out4[1] = m.pad[1];
    out4[2] = m.pad[2] & 0xfffff;
    out4[3] = m.pad[2] >> 20;
    return TWG_OK;
}

TWG_API int64_t twg_kernel_launches(const twg_ctx* c) { return c ? c->launches : 0; }

TWG_API twg_status twg_profile(twg_ctx* c, int32_t enable) {
    TWG_NVTX("twg_profile");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    c->prof = enable != 0;
    c->ev_used = 0;
    c->prof_launches = 0;
    c->prof_cells = 0;
    c->prof_ms = 0.0;
    return TWG_OK;
}

TWG_API twg_status twg_profile_read(twg_ctx* c, double* relax_ms, int64_t* relax_launches, int64_t* cell_sweeps) {
    TWG_NVTX("twg_profile_read");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    double ms = 0.0;
    for (int q = 0; q + 1 < c->ev_used; q += 2) {
        float e = 0.f;
        TWG_CUDA(c, cudaEventElapsedTime(&e, c->ev_pool[q], c->ev_pool[q + 1]));
        ms += e;
    }
    if (relax_ms) *relax_ms = ms;
    if (relax_launches) *relax_launches = c->prof_launches;
    if (cell_sweeps) *cell_sweeps = c->prof_cells;
    return TWG_OK;
}

TWG_API const char* twg_last_error(const twg_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

