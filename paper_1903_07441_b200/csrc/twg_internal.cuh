// twg_internal.cuh -- context layout, kernel argument structs and sm_100a PTX helpers
// shared by the libtwg.so translation units (product path only; the CPU
// oracle under oracle/ shares nothing with this file).
#pragma once

#include <cuda.h>  // CUtensorMap (driver types only; the encode entry point is fetched at runtime)
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "../../include/twg.h"

namespace twg {

// ---------------------------------------------------------------- relaxation tiling
// One warp owns a vertical strip of kStripW = 128 cells (4 per lane, one float4)
// and `hseg` output rows.  Rows stream through a per-warp TMA ring of kStages
// stages of NW = 2T + 2 rows (one TMA box = one unrolled block of the row loop);
// the 2T half-sweeps of T red-black sweeps run as a register wavefront
// (DESIGN.md "k_rb_tblock").
#ifndef TWG_RELAX_WARPS
#define TWG_RELAX_WARPS 8
#endif
constexpr int kWarpsPerCta = TWG_RELAX_WARPS;  // 8: one CTA per SM at T = 6 (198 registers)
constexpr int kStripW = 128;
#ifndef TWG_RELAX_STAGES
#define TWG_RELAX_STAGES 3
#endif
constexpr int kStages = TWG_RELAX_STAGES;
constexpr int kMaxT = 8;
constexpr int kMaxLocalSlabs = 16;  // slabs of one local row-slab group

__host__ __device__ constexpr int halo_cols(int T) { return 4 * ((2 * T + 3) / 4); }  // round_up(2T, 4)
__host__ __device__ constexpr int out_cols(int T) { return kStripW - 2 * halo_cols(T); }

struct RelaxArgs {
    float* u0;           // ping-pong buffer 0, scenario 0
    float* u1;           // ping-pong buffer 1, scenario 0
    const int* cur;      // per-scenario buffer index holding the field at twg_relax entry
    int lp;              // launch parity: this launch reads buffer cur[b] ^ lp, writes the other
    int64_t P;           // pitch (floats)
    int64_t sstride;     // scenario stride (floats)
    int W, H;
    int n_strips, hseg;
    int seg_begin, seg_end;  // launched segment range
    int row_lo, row_hi;  // output rows of this launch: segment s covers [row_lo + s hseg, ...) within row_hi
    int res_r0, res_r1;  // rows whose cells count in the residual (owned rows of a slab)
    const int* done;     // per-scenario done flags
    unsigned* res;       // per-scenario residual (float bits, atomicMax), used when RESID
    const int4* fixbox;  // [B][2] boxes (x0, x1, y0, y1) of the positive fixed cells: goal, imported field
    int force_slow;      // 1: every warp takes the scalar path (TWG_RELAX_SLOW=1, tests)
};

// Per-scenario parameters of one encode (rows a1-a3), built on the host.
struct ScenParams {
    double xr, yr, c, s, speed;  // robot position, cos/sin(theta) (host libm), speed
    int b;                       // scenario index
    int gx, gy;                  // goal cell
    int rcx, rcy;                // robot cell
    int old_gx, old_gy;          // previous goal (-1: none)
    int warm;
    int cur;                     // buffer index holding the scenario's field
    int n_tracks;
    int n_prev_boxes;
    int64_t track_off;           // first track of this scenario in EncodeArgs::src
};

struct WarpCfgDev {
    double dt, Q[16], w, eps_v, rs;
    int hmax;
    int hmode;  // 0: Eq. 16 (C18); 1: ring time (C26)
    int fmode;  // 0: predicted covariance (C19); 1: posterior covariance (C27)
};

struct TrkReq {  // one scenario of a tracker tick (row f1)
    int b;            // scenario
    int n, m;         // tracks before the tick, detections
    int limit;        // track capacity after the tick
    int64_t det_off;  // first detection in TrackArgs::det
};

// Speculative segment walkers (k_walk, row a7): sample cells of the previous path become markers
// in the direction bytes, and one walker per marker runs concurrently with the walker from the robot.
constexpr int kSpecMax = 64;     // segment walkers per scenario
constexpr int kSpecMinSeg = 32;  // minimum previous-path cells between two markers
constexpr int kSpecMaxB = 4;     // contexts with at most this many scenarios speculate
constexpr int kDirMarker = 8;    // direction byte of marker k: kDirMarker + k

struct SpecTab {  // per scenario: pos / K by k_spec_stitch (next walk's samples), orig by k_index_dir
    int K;                // samples (sample k at cell (k + 1) S of the previous walk)
    int pad;
    int2 pos[kSpecMax];   // marker cell, (-1, -1) when the sample was out of grid or a duplicate
    int orig[kSpecMax];   // the direction byte the marker replaced, -1 until placed (restored by k_spec_stitch)
};

struct SegOut {  // per walker (0: from the robot, 1 + k: from marker k)
    int state;   // 1 goal, 2 no path (obstacle, no neighbour, > max_len), 3 reached a marker
    int n;       // cells counted from the walker's start cell (inclusive) to its end cell (inclusive)
    int next;    // state 3: the marker reached
    int pad;
};

struct PathMeta {  // per scenario, written by k_walk / k_band
    int n_cells;
    int status;
    int n_smooth;
    float next_x, next_y;
    int pad[3];
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TWG_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TWG_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 3D TMA tile load (global -> shared), completion signalled on `bar` (complete_tx).
// Out-of-bounds elements (negative or >= extent coordinates) are zero-filled,
// i.e. +0.0f = fixed obstacle, which is the grid-boundary condition (C4).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Field encoding (include/twg.h): free = sign bit set (value -u), fixed = sign clear.
// Programmatic dependent launch (sm_90+): a kernel of the relaxation chain is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so it is launched while the previous kernel
// drains.  pdl_wait: before touching anything the previous kernel wrote.  pdl_trigger: once this
// CTA has issued its last work, so the successor's CTAs are only scheduled when every CTA of this
// grid is finishing (triggering at the start lets early successor CTAs crowd some SMs and
// unbalances the launch).  Without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Small kernels of the encode and path chains: wait, then let the successor be scheduled at once.
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}

// True the first time it is called for the current device (per-device one-time set-up of kernel
// attributes and module loading; a process may hold contexts on several devices).
inline bool first_on_device(unsigned long long& mask) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    if (mask & bit) return false;
    mask |= bit;
    return true;
}

__device__ __forceinline__ bool is_free(float v) { return __float_as_int(v) < 0; }

// Device-side bounds checks of the checked build (-DTWG_CHECKED, tests/test_gpu_checked.py): the
// substitute for compute-sanitizer's memcheck where the GPU pool does not run it.  A failed check
// prints its location and traps (the launch fails with cudaErrorLaunchFailure); compiled out otherwise.
#ifdef TWG_CHECKED
#define TWG_CHECK(cond)                                                                                   \
    do {                                                                                                  \
        if (!(cond)) {                                                                                    \
            printf("TWG_CHECK failed: %s at %s:%d (block %d,%d thread %d)\n", #cond, __FILE__, __LINE__,  \
                   (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                                    \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define TWG_CHECK(cond) \
    do {                \
    } while (0)
#endif

}  // namespace twg

// ---------------------------------------------------------------- context
struct twg_ctx {
    static constexpr int kMaxT = twg::kMaxT;
    int device = 0;
    int n_sm = 148;
    cudaStream_t stream = nullptr;
    int W = 0, H = 0, B = 0, row_off = 0, ghost = 0;
    double cs = 0.1, ox = 0.0, oy = 0.0;
    int64_t P = 0;        // pitch in floats
    int64_t sstride = 0;  // floats per scenario field
    float* u[2] = {nullptr, nullptr};
    std::vector<int> cur;          // per scenario: which buffer holds the current field
    int* d_ctl = nullptr;          // one allocation [7][B]: done, cur, sweeps, where, res bits, res, flags
    int* d_cur = nullptr;          // device copy used by the tile kernel
    CUtensorMap tmap[2][kMaxT + 1];  // [buffer][T]: box = 128 x (2T + 2) rows
    uint8_t* mask = nullptr;       // device [B][H][W]
    std::vector<uint8_t> hmask;    // host copy (validation only)
    // relaxation control, [B] each
    int* d_done = nullptr;
    int* d_sweeps = nullptr;
    unsigned* d_res_bits = nullptr;
    float* d_res = nullptr;
    int* d_where = nullptr;
    int* d_flags = nullptr;
    int4* d_fixbox = nullptr;      // [B][2]: goal box, imported-field box (k_rb_tblock's fast path)
    // encode state
    struct Scen {
        int gx = -1, gy = -1, rcx = -1, rcy = -1;
        double rx = 0.0, ry = 0.0;  // robot position of the last encode (m): the global robot cell of a slab
        int n_tracks = 0, n_boxes = 0;
        int trk_n = 0;  // tracks in the resident tracker table (row f1)
        bool encoded = false, static_dirty = true;
    };
    std::vector<Scen> scen;
    int track_cap = 0;                 // per scenario
    twg_track* d_tracks = nullptr;     // [B][cap]
    int* d_t = nullptr;                // [B][cap]
    int* d_j = nullptr;
    double* d_pred = nullptr;          // [B][cap][3]
    int4* d_boxes = nullptr;           // [B][cap] (x0, x1, y0, y1) inclusive; empty if x0 > x1
    int* d_missed = nullptr;           // [B][cap] tracker missed counters (row f1)
    // tracker scratch (row f1)
    int trk_scratch_cap = 0;           // per-scenario capacity of the [B][cap] scratch tables
    twg_track* d_trk_pred = nullptr;
    int* d_trk_misn = nullptr;
    int* d_trk_match = nullptr;
    int trk_mcap = 0, trk_pcap = 0, trk_nreq_cap = 0;
    uint8_t* d_trk_used = nullptr;     // [nreq][mcap]
    ulonglong2* d_trk_pairs = nullptr; // [nreq][pcap]
    int* d_trk_ctl = nullptr;          // [3][nreq]: pair count, flags, tracks out
    twg::TrkReq* d_trk_req = nullptr;
    double2* d_trk_det = nullptr;
    int64_t trk_det_cap = 0;
    // lexicographic relaxation (f3)
    int lex_tx = 0, lex_ty = 0;
    std::vector<std::pair<int, int2*>> lex_lists;  // task lists per launch length
    int* d_lex_tdone = nullptr;
    unsigned* d_lex_task = nullptr;
    // closed-loop simulator (row f2)
    int sim_ocap = 0;
    double* d_sim_rob = nullptr;       // [B][6]
    int* d_sim_int = nullptr;          // [2][B]: ticks, status
    double* d_sim_goal = nullptr;      // [B][2]
    int* d_sim_nobs = nullptr;         // [B]
    double* d_sim_obs = nullptr;       // [B][ocap][4]
    double* d_sim_obs_old = nullptr;   // [B][ocap][4]
    double* d_sim_speed = nullptr;     // [B][ocap]
    double2* d_sim_det = nullptr;      // [B][ocap]
    int* d_sim_hist = nullptr;         // [B][36]
    std::vector<double> sim_rob;       // host mirror [B][6]
    std::vector<int> sim_ticks, sim_status, sim_nobs;
    twg::ScenParams* d_params = nullptr;  // inside the parameter block (after d_wcfg)
    unsigned char* d_param_block = nullptr;
    int params_cap = 0;
    twg::WarpCfgDev* d_wcfg = nullptr;
    int* d_track_off = nullptr;        // scatter offsets + scenario indices of one encode call
    twg_track* d_track_tmp = nullptr;  // contiguous device copy of host track input
    int64_t track_tmp_cap = 0;
    int track_off_cap = 0;
    // path buffers
    int path_len_cap = 0, smooth_cap = 0;
    int2* d_cells = nullptr;           // [B][path_len_cap]
    float2* d_wp = nullptr;            // [B][path_len_cap]
    float2* d_smooth = nullptr;        // [B][smooth_cap]
    twg::PathMeta* d_meta = nullptr;   // [B]
    twg::SpecTab* d_spec = nullptr;    // [B] markers of the speculative walk (B <= kSpecMaxB)
    twg::SegOut* d_seg = nullptr;      // [B][kSpecMax + 1] walker results
    int2* d_seg_cells = nullptr;       // [B][kSpecMax][path_len_cap + 1] segment cells
    uint8_t* d_dir = nullptr;          // index matrix (direction bytes) [B][H][P]
    std::vector<int> cur_cache, part_cache;  // cur / participation as last uploaded (twg_relax)
    CUtensorMap dir_map;               // TMA view of d_dir for the walker's windows
    // pinned host staging
    void* h_stage = nullptr;
    size_t h_stage_bytes = 0;
    size_t stage_off = 0;
    // row-slab sharding: this context holds slab `rank` of `nranks` of a global grid of
    // H_global rows, owned global rows [r0, r1) plus ghost = 2k rows per side (row_off = r0 - 2k)
    struct Shard {
        int nranks = 1, rank = 0, k = 0;  // k: sweeps between ghost exchanges
        int H_global = 0, r0 = 0, r1 = 0;
        void* nccl = nullptr;             // ncclComm_t of an NCCL group (not owned)
        std::vector<twg_ctx*> peers;      // local group (one process), rank order; empty otherwise
        cudaStream_t comm = nullptr;      // boundary bands, exchange and residual max
        cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
        std::shared_ptr<void> streams;    // owner of comm / ev (shared by the slabs of a local group)
    } shard;
    bool sharded() const { return shard.nccl != nullptr || !shard.peers.empty(); }
    // accounting
    int64_t launches = 0;
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    int ev_used = 0;
    int64_t prof_launches = 0, prof_cells = 0;
    double prof_ms = 0.0;
    std::string err;
};
