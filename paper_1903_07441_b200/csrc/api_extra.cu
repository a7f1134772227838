// api_extra.cu -- row f3 exports (full index matrix, per-cell warp map) and the slab walk hand-over.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "api_host.cuh"

using namespace twg;
using namespace twg::host;

TWG_API twg_status twg_walk_from(twg_ctx* c, int32_t b, int32_t x, int32_t y, int32_t max_cells, int32_t* cells_xy,
                                 int32_t* n_cells, int32_t* code, int32_t* next_xy) {
    TWG_NVTX("twg_walk_from");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (b < 0 || b >= c->B || x < 0 || x >= c->W || y < c->ghost || y >= c->H - c->ghost || max_cells < 0 || !code)
        return fail(c, TWG_E_INVALID_ARG, "bad argument (the start must lie in the owned rows)");
    int* d = nullptr;
    TWG_CUDA(c, cudaMallocAsync(reinterpret_cast<void**>(&d), (4 + 2 * (size_t)std::max(max_cells, 1)) * sizeof(int),
                                c->stream));
    const float* f = c->u[c->cur[b]] + (int64_t)b * c->sstride;
    TWG_CUDA(c, launch_walk_from(f, c->P, c->W, c->H, c->ghost, c->H - c->ghost, x, y, max_cells, d + 4, d, c->stream));
    c->launches += 1;
    int h[4];
    TWG_CUDA(c, cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    if (cells_xy && h[1] > 0)
        TWG_CUDA(c, cudaMemcpy(cells_xy, d + 4, (size_t)h[1] * 2 * sizeof(int), cudaMemcpyDeviceToHost));
    TWG_CUDA(c, cudaFreeAsync(d, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    *code = h[0];
    if (n_cells) *n_cells = h[1];
    if (next_xy) {
        next_xy[0] = h[2];
        next_xy[1] = h[3];
    }
    return TWG_OK;
}

// Shared by twg_index_matrix and twg_band_index: Eq. 3 for every cell of scenario b into d_dir.
static twg_status index_matrix_core(twg_ctx* c, int32_t b) {
    twg_status st = ensure_params(c, 1);
    if (st != TWG_OK) return st;
    ScenParams sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.b = b;
    sp.cur = c->cur[b];
    void* hp = nullptr;
    TWG_CUDA(c, stage_alloc(c, sizeof(ScenParams), &hp));
    std::memcpy(hp, &sp, sizeof(sp));
    TWG_CUDA(c, cudaMemcpyAsync(c->d_params, hp, sizeof(ScenParams), cudaMemcpyHostToDevice, c->stream));
    PathArgs p;
    std::memset(&p, 0, sizeof(p));
    p.u0 = c->u[0];
    p.u1 = c->u[1];
    p.P = c->P;
    p.sstride = c->sstride;
    p.W = c->W;
    p.H = c->H;
    p.params = c->d_params;
    p.nscen = 1;
    p.dir = c->d_dir;
    p.istride = c->sstride;
    TWG_CUDA(c, launch_index_dir(p, c->stream));
    c->launches += 1;
    return TWG_OK;
}

TWG_API twg_status twg_band_index(twg_ctx* c, int32_t b, const twg_band_cfg* cfg, uint8_t* out, int32_t* cells_xy,
                                  int32_t* n_cells) {
    TWG_NVTX("twg_band_index");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!cfg || b < 0 || b >= c->B || cfg->iterations < 0 || cfg->max_len < 1)
        return fail(c, TWG_E_INVALID_ARG, "bad argument");
    if (c->ghost > 0) return fail(c, TWG_E_INVALID_ARG, "the per-cell band is not available on a row slab");
    const twg_ctx::Scen& sc = c->scen[b];
    if (!sc.encoded) return fail(c, TWG_E_INVALID_ARG, "twg_band_index before set_obstacles");
    st = index_matrix_core(c, b);
    if (st != TWG_OK) return st;
    uint8_t* dir = c->d_dir + (int64_t)b * c->sstride;
    const float* f = c->u[c->cur[b]] + (int64_t)b * c->sstride;
    int nl = 0;
    TWG_CUDA(c, launch_cellband(f, c->P, c->W, c->H, dir, cfg->iterations, cfg->k_t, &nl, c->stream));
    c->launches += nl;
    if (out)
        TWG_CUDA(c, cudaMemcpy2DAsync(out, c->W, dir, c->P, c->W, c->H, cudaMemcpyDefault, c->stream));
    int* d = nullptr;
    TWG_CUDA(c, cudaMallocAsync(reinterpret_cast<void**>(&d), (2 + 2 * (size_t)cfg->max_len) * sizeof(int), c->stream));
    TWG_CUDA(c, launch_walk_dir(dir, c->P, sc.rcx, sc.rcy, cfg->max_len, d, reinterpret_cast<int2*>(d + 2), c->stream));
    c->launches += 1;
    int h[2];
    TWG_CUDA(c, cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    if (cells_xy && h[1] > 0)
        TWG_CUDA(c, cudaMemcpy(cells_xy, d + 2, (size_t)h[1] * 2 * sizeof(int), cudaMemcpyDeviceToHost));
    TWG_CUDA(c, cudaFreeAsync(d, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    if (n_cells) *n_cells = h[1];
    if (h[0] != TWG_OK) return fail(c, TWG_E_NO_PATH, "no path along the optimised index matrix");
    return TWG_OK;
}

TWG_API twg_status twg_index_matrix(twg_ctx* c, int32_t b, uint8_t* out) {
    TWG_NVTX("twg_index_matrix");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!out || b < 0 || b >= c->B) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    st = index_matrix_core(c, b);
    if (st != TWG_OK) return st;
    // [H][P] -> [H][W] (cudaMemcpyDefault: out may be host or device)
    TWG_CUDA(c, cudaMemcpy2DAsync(out, c->W, c->d_dir + (int64_t)b * c->sstride, c->P, c->W, c->H, cudaMemcpyDefault,
                                  c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

TWG_API twg_status twg_warp_map(twg_ctx* c, const twg_robot* robot, double warp_spacing, int32_t* out) {
    TWG_NVTX("twg_warp_map");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!out || !robot || !(warp_spacing > 0.0)) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    const double cth = std::cos(robot->theta), sth = std::sin(robot->theta);  // host libm (C25)
    const size_t bytes = (size_t)c->W * c->H * sizeof(int32_t);
    int32_t* dst = out;
    if (!is_device_ptr(out)) TWG_CUDA(c, cudaMallocAsync(reinterpret_cast<void**>(&dst), bytes, c->stream));
    TWG_CUDA(c, launch_warp_map(dst, c->W, c->H, c->cs, c->ox, c->oy, robot->x, robot->y, cth, sth, warp_spacing,
                                c->stream));
    c->launches += 1;
    if (dst != out) {
        TWG_CUDA(c, cudaMemcpyAsync(out, dst, bytes, cudaMemcpyDeviceToHost, c->stream));
        TWG_CUDA(c, cudaFreeAsync(dst, c->stream));
    }
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

