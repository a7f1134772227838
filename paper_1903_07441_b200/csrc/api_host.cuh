// api_host.cuh -- host-side helpers shared by the C ABI translation units (host_core.cu, api*.cu).
#pragma once
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX 3

#include "twg_kernels.cuh"

// NVTX range for the lifetime of a scope (one per C-ABI call and per phase of a plan step), so that
// nsys / ncu --nvtx attribute device work to the call that enqueued it (tracing).
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};
#define TWG_NVTX_CAT2(a, b) a##b
#define TWG_NVTX_CAT(a, b) TWG_NVTX_CAT2(a, b)
#define TWG_NVTX(name) twg::host_nvtx::NvtxScope TWG_NVTX_CAT(twg_nvtx_, __LINE__)(name)

namespace twg {
namespace host_nvtx {
using ::NvtxScope;
}
namespace host {

extern std::string g_create_err;  // message of the last failed twg_create

twg_status fail(twg_ctx* c, twg_status st, const std::string& msg);

#define TWG_CUDA(ctx, expr)                                                                                 \
    do {                                                                                                    \
        cudaError_t e_ = (expr);                                                                            \
        if (e_ != cudaSuccess)                                                                              \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? TWG_E_NO_MEMORY : TWG_E_CUDA,                \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                                \
    } while (0)

template <class T>
cudaError_t dev_alloc(T** p, size_t n) {
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T));
}

bool is_device_ptr(const void* p);
bool make_tmap(CUtensorMap* m, float* base, int W, int H, int B, int64_t P, int rows);
bool make_dir_map(CUtensorMap* m, uint8_t* base, int H, int B, int64_t P);
// Pinned staging ring for host->device copies (synchronises the stream when it wraps).
cudaError_t stage_alloc(twg_ctx* c, size_t bytes, void** out);
twg_status ensure_track_cap(twg_ctx* c, int cap);
twg_status ensure_params(twg_ctx* c, int n);
twg_status ensure_path_cap(twg_ctx* c, int max_len, int max_smooth);
twg_status check_ctx(twg_ctx* c);

struct EncodeReq {
    int b;
    twg_robot robot;
    int gx, gy;
    int n;
    int64_t track_off;  // offset into the caller's track array
};

twg_status validate(twg_ctx* c, const EncodeReq& r, int* rcx, int* rcy);
// Rows a1-a3 for a list of scenarios (resident: use the tracker tables already in d_tracks).
twg_status encode(twg_ctx* c, const std::vector<EncodeReq>& reqs, const twg_track* tracks, const twg_warp_cfg* wc,
                  int warm_req, bool resident = false);
// Rows a4-a6 for the scenarios with part[b] != 0 (a context of a local slab group relaxes the group).
twg_status relax(twg_ctx* c, const twg_relax_cfg* cfg, const std::vector<int>& part, int* sweeps_done,
                 float* residual);
twg_status relax_group(const std::vector<twg_ctx*>& g, const twg_relax_cfg* cfg, const std::vector<int>& part,
                       int* sweeps_done, float* residual);

// NCCL (nccl_link.cu): resolved at run time from the libnccl.so.2 already loaded by the process
// (torch's), else loaded by name; every call reports TWG_E_NCCL through fail() on error.
twg_status nccl_load(twg_ctx* c);
twg_status nccl_comm_rank(twg_ctx* c, void* comm, int* rank, int* nranks);
// One group call: send s_up (cnt floats) to `up` and receive r_up from it, the same with `dn`
// (-1: no such neighbour).
twg_status nccl_exchange(twg_ctx* c, size_t cnt, int up, int dn, const float* s_up, float* r_up, const float* s_dn,
                         float* r_dn, cudaStream_t st);
twg_status nccl_allreduce_max_u32(twg_ctx* c, unsigned* buf, int n, cudaStream_t st);
twg_status nccl_bcast_i32(twg_ctx* c, int* buf, int n, int root, cudaStream_t st);
twg_status nccl_allreduce_sum_u32(twg_ctx* c, unsigned* buf, size_t n, cudaStream_t st);
// Rows a7-a9 on a row-slab group (api_shard.cu): walk handed over between the slabs, then the band on
// the gathered corridor rows; every slab returns the whole path (global cells).
twg_status sharded_extract_path(twg_ctx* c, const twg_band_cfg* cfg, int32_t* cells_xy, int32_t* n_cells,
                                float* smooth_xy, int32_t* n_smooth, float* next_xy);
// Rows a7-a9 for a list of scenarios (results stay on the device).
twg_status path(twg_ctx* c, const std::vector<int>& bs, const twg_band_cfg* cfg);
// Row f1 tick for the requests rq (det_off relative to `det`, a device array of (x, y) pairs).
twg_status track_core(twg_ctx* c, std::vector<TrkReq> rq, const double2* det, const twg_warp_cfg* wc,
                      const twg_tracker_cfg* cfg, std::vector<int>& n_out);

}  // namespace host
}  // namespace twg
