// twg_kernels.cuh -- host launchers of the libtwg.so kernels (product path).
#pragma once
#include "twg_internal.cuh"

namespace twg {

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


// k_relax.cu (rows a4-a6)
cudaError_t launch_rb_tblock(int T, const CUtensorMap& map0, const CUtensorMap& map1, const RelaxArgs& a, int B, int qoff, bool resid,
                             cudaStream_t st);
int rb_tblock_ctas_per_sm(int T);  // CTAs of k_rb_tblock<T> resident per SM (occupancy)
cudaError_t launch_jacobi(const RelaxArgs& a, int B, bool resid, cudaStream_t st);
struct LexArgs {
    float* u0;
    float* u1;
    const int* cur;
    int64_t P, sstride;
    int W, H, B;
    int TX, TY, ntiles;    // 32 x 32 tiles
    const int2* tasks;     // [ntasks] (i | s << 16, j) in wavefront-time order (diag + 2 s)
    int ntasks;            // sweeps * ntiles
    int sweeps, base;      // sweeps in this launch; sweeps finished before it (this twg_relax call)
    int* tdone;            // [B][ntiles] sweeps finished per tile
    unsigned* task;        // task counter (zeroed before the launch)
    const int* done;
    unsigned* res;         // residual bits of the launch's last sweep (nullptr: not tracked)
    int res_r0, res_r1;
};
cudaError_t launch_lex(const LexArgs& a, int n_sm, cudaStream_t st);
cudaError_t launch_warp_map(int32_t* out, int W, int H, double cs, double ox, double oy, double xr, double yr, double c,
                            double s, double w, cudaStream_t st);
bool small_grid(int W, int H);  // k_rb_small applies (the field fits in shared memory)
cudaError_t launch_rb_small(const RelaxArgs& a, int B, int max_sweeps, int check_every, float tol, int qoff,
                            int* sweeps_out, float* res_out, cudaStream_t st);
cudaError_t launch_res_group_max(unsigned* const* ptrs, int n, int B, cudaStream_t st);
cudaError_t launch_relax_init(int* done, int* sweeps, int* where, unsigned* res_bits, float* res, int B, cudaStream_t st);
cudaError_t launch_check(int B, int* done, int* sweeps, unsigned* res_bits, float* res_final, int* where, int chunk,
                         int check_every, int max_sweeps, float tol, const int* cur, int lp, cudaStream_t st);
cudaError_t launch_init_field(float* u, int64_t P, int64_t sstride, int W, int H, int B, cudaStream_t st);
cudaError_t launch_convert(const float* src, int64_t P, int W, int H, float* dst, int mode, cudaStream_t st);
cudaError_t launch_import(const float* src, int W, int H, float* dst, int64_t P, int4* box, cudaStream_t st);
cudaError_t launch_fixup(float* u0, float* u1, int64_t sstride, int B, const int* where, const int* cur, int lp,
                         cudaStream_t st);

// k_stamp.cu (rows a1-a3)
struct EncodeArgs {
    float* u0;             // ping-pong buffers, scenario 0 (ScenParams::cur selects)
    float* u1;
    int64_t P, sstride;
    int W, H;
    const uint8_t* mask;   // [B][H][W]
    const ScenParams* params;  // [nscen]
    int nscen;
    const WarpCfgDev* wcfg;
    twg_track* tracks;         // [B][cap] (the resident track table)
    const twg_track* src;      // caller's tracks (copied into `tracks` by k_track_predict), or nullptr
    int* missed;               // [B][cap] tracker miss counters, reset for copied tracks
    int cap;
    int* t_out;            // [B][cap]
    int* j_out;
    double* pred;          // [B][cap][3]
    int4* boxes;           // [B][cap]
    int* flags;            // [B] warning flags
    int4* fixbox;          // [B][2]: goal box (set with the goal), imported-field box (cleared by a cold encode)
    double cs, ox, oy;
};
cudaError_t launch_encode(const EncodeArgs& e, int max_prev_boxes, int max_tracks, int any_cold, int* n_launch,
                          cudaStream_t st);


// k_track.cu (row f1: tracker tick)
enum : int { kTrkTruncated = 1, kTrkSingular = 2, kTrkOverflow = 4 };
struct TrackArgs {
    twg_track* trk;        // [B][cap] resident table (= the encode track table)
    int* missed;           // [B][cap]
    twg_track* pred;       // [B][cap] scratch
    int* mis_new;          // [B][cap] scratch
    int* match;            // [B][cap] detection matched to each track, or -1
    uint8_t* used;         // [nreq][mcap] detection matched
    const double2* det;    // concatenated detections (x, y)
    const TrkReq* req;     // [nreq]
    ulonglong2* pairs;     // [nreq][pcap] gated pairs (d^2 bits, track << 32 | detection)
    int* pcount;           // [nreq]
    int* flags;            // [nreq]
    int* n_out;            // [nreq]
    int cap, mcap, pcap;   // pcap: power of two
    int prune_after;
    double Q[16], dt, r2, gate2, var_pos, var_vel;
};
cudaError_t launch_track_step(const TrackArgs& t, int nreq, int max_n, int max_m, int* n_launch, cudaStream_t st);

// k_path.cu (rows a7-a9)
struct PathArgs {
    const float* u0;       // ping-pong buffers, scenario 0 (ScenParams::cur selects)
    const float* u1;
    int64_t P, sstride;
    int W, H;
    const ScenParams* params;  // robot/goal cells per entry
    int nscen;
    int max_len, max_smooth, iters;
    float step, kt;
    int2* cells;           // [B][max_len_cap]
    float2* wp;            // [B][max_len_cap]
    float2* smooth;        // [B][smooth_cap]
    int len_cap, smooth_cap;
    PathMeta* meta;        // [B]
    uint8_t* dir;          // index matrix M_idx as one direction byte per cell, [B][H][P]
    int64_t istride;       // entries per scenario (H * P)
    CUtensorMap dir_map;   // M_idx as a 2D {P, H * B} uint8 tensor, box {256, 176} (k_walk windows)
    SpecTab* spec;         // [B] (spec_on)
    SegOut* seg;           // [B][kSpecMax + 1] (spec_on)
    int2* seg_cells;       // [B][kSpecMax][len_cap + 1] (spec_on)
    int spec_on;           // speculative segment walkers (markers in k_index_dir / k_walk / k_spec_stitch)
};
cudaError_t launch_path(const PathArgs& p, int* n_launch, cudaStream_t st);
cudaError_t launch_band_resample(const PathArgs& p, cudaStream_t st);  // a8-a9 after a walk (2 launches)
cudaError_t launch_seg_append(const int* seg, const int* wout, int row_off, int at, int2* path, int* msg,
                              cudaStream_t st);
cudaError_t launch_cells_shift(const int2* in, int n, int dy, int2* out, cudaStream_t st);
cudaError_t launch_index_dir(const PathArgs& p, cudaStream_t st);  // k_index_dir alone (twg_index_matrix)
// f3 per-cell band on the index matrix (2 iters launches) and the walk along a matrix
cudaError_t launch_cellband(const float* f, int64_t P, int W, int H, uint8_t* dir, int iters, float kt, int* n_launch,
                            cudaStream_t st);
cudaError_t launch_walk_dir(const uint8_t* dir, int64_t P, int x, int y, int max_len, int* out, int2* cells,
                            cudaStream_t st);
cudaError_t launch_walk_from(const float* f, int64_t P, int W, int H, int r0, int r1, int x, int y, int max_cells,
                             int* cells, int* out, cudaStream_t st);

// k_sim.cu (row f2: closed-loop simulator)
struct SimArgs {
    int B, W, H, ocap;
    double cs, ox, oy;
    const uint8_t* mask;     // [B][H][W]
    double* rob;             // [B][6]: x, y, hx, hy, speed, length
    int* ticks;              // [B]
    int* status;             // [B]: 0 running, 1 success, 2 collision, 3 timeout, 4 idle
    const double* goal;      // [B][2] goal centre (m)
    const int* n_obs;        // [B]
    double* obs;             // [B][ocap][4]: x, y, vx, vy
    double* obs_old;         // [B][ocap][4] scratch
    const double* obs_speed; // [B][ocap]
    double2* det;            // [B][ocap] detections of the current tick
    int* hist;               // [B][36] turning-angle histogram (5 degree bins)
    const PathMeta* meta;    // [B] this tick's plan (walk status, next waypoint)
    double dt, r_robot, r_obs, goal_r, turn_dist, sigma_h, sigma_z, cos_d, sin_d;
    double cos_bins[37];
    uint64_t seed;
    int max_ticks;
};
cudaError_t launch_sim_move(const SimArgs& a, cudaStream_t st);
cudaError_t launch_sim_sense(const SimArgs& a, int only, cudaStream_t st);

// Module preloading (called once by twg_create)
void preload_relax_kernels();
void preload_stamp_kernels();
void preload_path_kernels();
void preload_track_kernels();
void preload_sim_kernels();

}  // namespace twg
