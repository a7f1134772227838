// api_shard.cu -- rows a7-a9 on a row-slab group (SURVEY 8(e) "sharded path extraction hands the
// walker off between ranks").  The descent walk (Eq. 3, Alg. 1) runs on the slab
// owning the current cell until it steps into a ghost row; the walker (next cell, cells so far) is then
// handed to that neighbour (ncclBroadcast of 4 ints from the owner, or, for a local group, read on the
// host).  Each slab keeps its segments at their offsets in a zeroed global path buffer, and a sum
// all-reduce gives every slab the whole path.  The rubber band (Eqs. 4-6) and the resampling need the
// field around the path: the rows [ymin - R, ymax + R] of the global grid (R bounds how far a waypoint
// and its bilinear stencil can move in I iterations of step s: I s sqrt(2) + 3) are assembled from the
// slabs' owned rows (bit patterns summed into a zeroed buffer -- exact), and the unchanged band and
// resampling kernels run on that corridor on every slab, giving identical results everywhere.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "api_host.cuh"

namespace twg {
namespace host {

// Stream-ordered device scratch released on every exit path.
struct AsyncBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~AsyncBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

static int owner_of(const twg_ctx* c, int gy) {
    const int n = c->shard.nranks, H = c->shard.H_global;
    const int base = H / n, extra = H % n;
    for (int r = 0; r < n; ++r) {
        const int r0 = r * base + std::min(r, extra), r1 = r0 + base + (r < extra ? 1 : 0);
        if (gy >= r0 && gy < r1) return r;
    }
    return -1;
}

twg_status sharded_extract_path(twg_ctx* c, const twg_band_cfg* cfg, int32_t* cells_xy, int32_t* n_cells,
                                float* smooth_xy, int32_t* n_smooth, float* next_xy) {
    const bool nccl = c->shard.nccl != nullptr;
    std::vector<twg_ctx*> g = nccl ? std::vector<twg_ctx*>{c} : c->shard.peers;
    twg_ctx* c0 = g[0];
    cudaStream_t st = c->stream;
    for (twg_ctx* m : g)
        if (!m->scen[0].encoded) return fail(c, TWG_E_INVALID_ARG, "extract_path before set_obstacles");
    const twg_ctx::Scen& sc = c->scen[0];
    const int max_len = cfg->max_len;
    // global robot cell (every slab has the same pose) and its owner
    const double oy_global = c->oy - (double)c->row_off * c->cs;
    int x = (int)std::floor((sc.rx - c->ox) / c->cs);
    int gy = (int)std::floor((sc.ry - oy_global) / c->cs);
    if (x < 0 || x >= c->W || gy < 0 || gy >= c->shard.H_global)
        return fail(c, TWG_E_OUT_OF_BOUNDS, "robot cell outside the grid");
    int owner = owner_of(c, gy);
    // device scratch: [msg 4 | walk out 4 | segment cells 2 max_len | path 2 max_len]
    AsyncBuf db;
    db.st = st;
    const size_t nints = 8 + 4 * (size_t)max_len;
    TWG_CUDA(c, cudaMallocAsync(&db.p, nints * sizeof(int), st));
    int* d = static_cast<int*>(db.p);
    TWG_CUDA(c, cudaMemsetAsync(d, 0, nints * sizeof(int), st));
    int* msg = d;
    int* wout = d + 4;
    int* seg = d + 8;
    int2* path = reinterpret_cast<int2*>(d + 8 + 2 * (size_t)max_len);
    int total = 0, code = TWG_E_NO_PATH;
    for (int hop = 0; hop <= 4 * c->shard.nranks + max_len; ++hop) {
        const int me = nccl ? c->shard.rank : owner;
        twg_ctx* w = nccl ? c : g[owner];
        if (me == owner) {
            const float* f = w->u[w->cur[0]];
            TWG_CUDA(c, launch_walk_from(f, w->P, w->W, w->H, w->ghost, w->H - w->ghost, x, gy - w->row_off,
                                         max_len - total, seg, wout, st));
            TWG_CUDA(c, launch_seg_append(seg, wout, w->row_off, total, path, msg, st));
            c->launches += 2;
        } else {
            TWG_CUDA(c, cudaMemsetAsync(msg, 0, 4 * sizeof(int), st));
        }
        if (nccl && c->shard.nranks > 1) {
            twg_status bs = nccl_bcast_i32(c, msg, 4, owner, st);
            if (bs != TWG_OK) return bs;
        }
        int h[4];
        TWG_CUDA(c, cudaMemcpyAsync(h, msg, sizeof(h), cudaMemcpyDeviceToHost, st));
        TWG_CUDA(c, cudaStreamSynchronize(st));
        code = h[0];
        total += h[3];
        if (code == TWG_OK || code == TWG_E_NO_PATH) break;
        owner += code == 1 ? -1 : 1;  // 1: the slab above, 2: the slab below
        x = h[1];
        gy = h[2];
        if (owner < 0 || owner >= c->shard.nranks) {
            code = TWG_E_NO_PATH;
            break;
        }
    }
    if (code != TWG_OK) {
        if (n_cells) *n_cells = 0;
        if (n_smooth) *n_smooth = 0;
        if (next_xy) {
            next_xy[0] = (float)x + 0.5f;
            next_xy[1] = (float)gy + 0.5f;
        }
        return fail(c, TWG_E_NO_PATH, "no path: the walk entered an obstacle or exceeded max_len");
    }
    if (nccl && c->shard.nranks > 1) {  // every slab wrote only its own segments: sum = the whole path
        twg_status rs = nccl_allreduce_sum_u32(c, reinterpret_cast<unsigned*>(path), 2 * (size_t)total, st);
        if (rs != TWG_OK) return rs;
    }
    std::vector<int2> hpath(total);
    TWG_CUDA(c, cudaMemcpyAsync(hpath.data(), path, (size_t)total * sizeof(int2), cudaMemcpyDeviceToHost, st));
    TWG_CUDA(c, cudaStreamSynchronize(st));
    int ymin = hpath[0].y, ymax = hpath[0].y;
    for (const int2& q : hpath) {
        ymin = std::min(ymin, q.y);
        ymax = std::max(ymax, q.y);
    }
    // the corridor: every row a waypoint or its 3 x 3 stencil can reach in I iterations of step s
    const int R = (int)std::ceil((double)cfg->iterations * std::fabs((double)cfg->step) * 1.41421356237) + 3;
    const int y0 = std::max(0, ymin - R), y1 = std::min(c->shard.H_global, ymax + R + 1);
    const int nrows = y1 - y0;
    const int64_t P = c->P;
    AsyncBuf cb;
    cb.st = st;
    TWG_CUDA(c, cudaMallocAsync(&cb.p, (size_t)nrows * P * sizeof(float), st));
    unsigned* corr = static_cast<unsigned*>(cb.p);
    TWG_CUDA(c, cudaMemsetAsync(corr, 0, (size_t)nrows * P * sizeof(float), st));
    for (twg_ctx* m : g) {  // owned rows of each slab inside [y0, y1)
        const int a = std::max(y0, m->shard.r0), e = std::min(y1, m->shard.r1);
        if (a >= e) continue;
        const float* src = m->u[m->cur[0]] + (int64_t)(a - m->row_off) * P;
        TWG_CUDA(c, cudaMemcpyAsync(corr + (int64_t)(a - y0) * P, src, (size_t)(e - a) * P * sizeof(float),
                                    cudaMemcpyDeviceToDevice, st));
    }
    if (nccl && c->shard.nranks > 1) {
        twg_status rs = nccl_allreduce_sum_u32(c, corr, (size_t)nrows * P, st);
        if (rs != TWG_OK) return rs;
    }
    // band + resampling on the corridor: cells with rows relative to y0, scenario 0 of a 1-scenario view
    twg_status es = ensure_path_cap(c0, max_len, cfg->max_smooth);
    if (es != TWG_OK) return es;
    es = ensure_params(c0, 1);
    if (es != TWG_OK) return es;
    TWG_CUDA(c, launch_cells_shift(path, total, -y0, c0->d_cells, st));
    ScenParams sp;
    std::memset(&sp, 0, sizeof(sp));
    PathMeta pm;
    std::memset(&pm, 0, sizeof(pm));
    pm.n_cells = total;
    pm.status = TWG_OK;
    char* hs = nullptr;
    TWG_CUDA(c, stage_alloc(c, 256 + sizeof(PathMeta), reinterpret_cast<void**>(&hs)));
    std::memcpy(hs, &sp, sizeof(sp));
    std::memcpy(hs + 256, &pm, sizeof(pm));
    TWG_CUDA(c, cudaMemcpyAsync(c0->d_params, hs, sizeof(sp), cudaMemcpyHostToDevice, st));
    TWG_CUDA(c, cudaMemcpyAsync(c0->d_meta, hs + 256, sizeof(pm), cudaMemcpyHostToDevice, st));
    PathArgs p;
    std::memset(&p, 0, sizeof(p));
    p.u0 = reinterpret_cast<const float*>(corr);
    p.u1 = reinterpret_cast<const float*>(corr);
    p.P = P;
    p.sstride = (int64_t)nrows * P;
    p.W = c->W;
    p.H = nrows;
    p.params = c0->d_params;
    p.nscen = 1;
    p.max_len = max_len;
    p.max_smooth = cfg->max_smooth;
    p.iters = cfg->iterations;
    p.step = cfg->step;
    p.kt = cfg->k_t;
    p.cells = c0->d_cells;
    p.wp = c0->d_wp;
    p.smooth = c0->d_smooth;
    p.len_cap = c0->path_len_cap;
    p.smooth_cap = c0->smooth_cap;
    p.meta = c0->d_meta;
    TWG_CUDA(c, launch_band_resample(p, st));
    c->launches += 3;
    PathMeta m;
    TWG_CUDA(c, cudaMemcpyAsync(&m, c0->d_meta, sizeof(m), cudaMemcpyDeviceToHost, st));
    TWG_CUDA(c, cudaStreamSynchronize(st));
    const int ns = std::min(m.n_smooth, cfg->max_smooth);
    if (smooth_xy && ns > 0) {
        TWG_CUDA(c, cudaMemcpyAsync(smooth_xy, c0->d_smooth, (size_t)ns * sizeof(float2), cudaMemcpyDeviceToHost, st));
        TWG_CUDA(c, cudaStreamSynchronize(st));
        for (int i = 0; i < ns; ++i) smooth_xy[2 * i + 1] += (float)y0;  // corridor rows -> global (exact)
    }
    if (cells_xy) std::memcpy(cells_xy, hpath.data(), (size_t)std::min(total, max_len) * sizeof(int2));
    if (n_cells) *n_cells = total;
    if (n_smooth) *n_smooth = m.n_smooth;
    if (next_xy) {
        next_xy[0] = m.next_x;
        next_xy[1] = m.next_y + (float)y0;
    }
    return m.n_smooth > cfg->max_smooth ? TWG_W_TRUNCATED : TWG_OK;
}

}  // namespace host
}  // namespace twg
