// Row f1: the tracker tick that precedes rows a1-a3 in Alg. 1's Map Update
// (P:680-688), batched over scenarios, fp64, resident on the device.
//
//   k_trk_predict   one thread per track: one Kalman predict (Eqs. 9-10, A of P:548-553) into a
//                   scratch table; resets the match/used flags
//   k_trk_pairs     32 x 32 (track, detection) tiles: squared distance of every pair, gated pairs
//                   appended to the request's pair list (warp-aggregated atomics)
//   k_trk_assoc     one CTA per request: sort the gated pairs by (d^2, track, detection) (bitonic,
//                   in shared memory up to 4096 pairs, else in the global list), then one thread
//                   takes them in order, keeping a pair iff both ends are still free -- the greedy
//                   "globally closest first" association of S:281-289 (C29)
//   k_trk_update    one thread per track: Eqs. 11-13 with H of P:558-565, R = sigma^2 I,
//                   P symmetrised (C28); missed counters
//   k_trk_compact   one CTA per request: prune (missed > prune_after), append one track per
//                   unmatched detection, capacity limit (C30)
//
// Bit-exactness with oracle/twg_oracle.c (orc_track_step): the same dense fp64 operation sequences
// (library compiled with -fmad=false) and the same tie order.
#include <algorithm>

#include "twg_kernels.cuh"

namespace twg {

// A x and A P A^T + Q, dense, k ascending (one step of Eqs. 9-10)
__device__ __forceinline__ void trk_predict1(const double* x, const double* P, const double* Q, double dt, double* xo,
                                             double* Po) {
    double A[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) A[q] = 0.0;
    A[0] = 1.0; A[5] = 1.0; A[10] = 1.0; A[15] = 1.0;
    A[2] = dt; A[7] = dt;
    double AP[16];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc = acc + A[r * 4 + k] * x[k];
        xo[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + A[r * 4 + k] * P[k * 4 + c];
            AP[r * 4 + c] = acc;
        }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + AP[r * 4 + k] * A[c * 4 + k];
            Po[r * 4 + c] = acc + Q[r * 4 + c];
        }
}

// Eqs. 11-13 with the explicit H; returns false (x, P untouched) if H P H^T + R is not
// positive definite.
__device__ __forceinline__ bool trk_kalman_update(double* x, double* P, double zx, double zy, double r2) {
    double Hm[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) Hm[q] = 0.0;
    Hm[0] = 1.0; Hm[5] = 1.0;
    const double R[4] = {r2, 0.0, 0.0, r2};
    const double z[2] = {zx, zy};
    double y[2], HP[8], S[4], Si[4], PHt[8], K[8], IKH[16], Pn[16], xn[4];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc = acc + Hm[r * 4 + k] * x[k];
        y[r] = z[r] - acc;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + Hm[r * 4 + k] * P[k * 4 + c];
            HP[r * 4 + c] = acc;
        }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + HP[r * 4 + k] * Hm[c * 4 + k];
            S[r * 2 + c] = acc + R[r * 2 + c];
        }
    const double det = S[0] * S[3] - S[1] * S[2];
    if (!(det > 0.0) || !(S[0] > 0.0) || !(det < 1.0e300)) return false;
    Si[0] = S[3] / det;
    Si[1] = -S[1] / det;
    Si[2] = -S[2] / det;
    Si[3] = S[0] / det;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + P[r * 4 + k] * Hm[c * 4 + k];
            PHt[r * 2 + c] = acc;
        }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 2; ++k) acc = acc + PHt[r * 2 + k] * Si[k * 2 + c];
            K[r * 2 + c] = acc;
        }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 2; ++k) acc = acc + K[r * 2 + k] * y[k];
        xn[r] = x[r] + acc;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 2; ++k) acc = acc + K[r * 2 + k] * Hm[k * 4 + c];
            IKH[r * 4 + c] = (r == c ? 1.0 : 0.0) - acc;
        }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + IKH[r * 4 + k] * P[k * 4 + c];
            Pn[r * 4 + c] = acc;
        }
#pragma unroll
    for (int r = 0; r < 4; ++r) x[r] = xn[r];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) P[r * 4 + c] = 0.5 * (Pn[r * 4 + c] + Pn[c * 4 + r]);
    return true;
}

__global__ void k_trk_predict(TrackArgs t) {
    const TrkReq& rq = t.req[blockIdx.y];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t tb = (int64_t)rq.b * t.cap;
    if (i < rq.n) {
        const twg_track tr = t.trk[tb + i];
        twg_track o;
        trk_predict1(tr.x, tr.P, t.Q, t.dt, o.x, o.P);
        t.pred[tb + i] = o;
        t.match[tb + i] = -1;
    }
    if (i < rq.m) t.used[(int64_t)blockIdx.y * t.mcap + i] = 0;
    if (i == 0) t.pcount[blockIdx.y] = 0;
}

constexpr int kPairTile = 32;

__global__ void __launch_bounds__(256) k_trk_pairs(TrackArgs t) {
    const TrkReq& rq = t.req[blockIdx.y];
    const int tiles_m = (rq.m + kPairTile - 1) / kPairTile;
    const int tiles = ((rq.n + kPairTile - 1) / kPairTile) * tiles_m;
    __shared__ double2 sp[kPairTile], sz[kPairTile];
    const int64_t tb = (int64_t)rq.b * t.cap;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int i0 = (tile / tiles_m) * kPairTile, j0 = (tile % tiles_m) * kPairTile;
        __syncthreads();
        if (threadIdx.x < kPairTile) {
            const int i = i0 + threadIdx.x;
            sp[threadIdx.x] = i < rq.n ? make_double2(t.pred[tb + i].x[0], t.pred[tb + i].x[1]) : make_double2(0, 0);
        } else if (threadIdx.x < 2 * kPairTile) {
            const int j = j0 + threadIdx.x - kPairTile;
            sz[threadIdx.x - kPairTile] = j < rq.m ? t.det[rq.det_off + j] : make_double2(0, 0);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kPairTile * kPairTile / 256; ++q) {
            const int e = q * 256 + threadIdx.x;
            const int ii = e / kPairTile, jj = e % kPairTile;
            const int i = i0 + ii, j = j0 + jj;
            bool keep = false;
            double d2 = 0.0;
            if (i < rq.n && j < rq.m) {
                const double dx = sz[jj].x - sp[ii].x;
                const double dy = sz[jj].y - sp[ii].y;
                d2 = dx * dx + dy * dy;
                keep = d2 <= t.gate2;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (bal) {
                const int lane = threadIdx.x & 31;
                int base = 0;
                if (lane == __ffs(bal) - 1) base = atomicAdd(&t.pcount[blockIdx.y], __popc(bal));
                base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
                if (keep) {
                    const int slot = base + __popc(bal & ((1u << lane) - 1u));
                    if (slot < t.pcap)
                        t.pairs[(int64_t)blockIdx.y * t.pcap + slot] =
                            make_ulonglong2((unsigned long long)__double_as_longlong(d2),
                                            ((unsigned long long)i << 32) | (unsigned)j);
                }
            }
        }
    }
}

__device__ __forceinline__ bool pair_less(const ulonglong2& a, const ulonglong2& b) {
    return a.x < b.x || (a.x == b.x && a.y < b.y);
}

// In-block bitonic sort of v[0, N) (N a power of two), ascending.
__device__ void bitonic_sort(ulonglong2* v, int N) {
    for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < N; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const ulonglong2 a = v[i], b = v[l];
                    const bool up = (i & k) == 0;
                    if (up ? pair_less(b, a) : pair_less(a, b)) {
                        v[i] = b;
                        v[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

constexpr int kSmemPairs = 4096;

__device__ __forceinline__ int block_scan(int v, int* sw, int* total);

__global__ void __launch_bounds__(1024) k_trk_assoc(TrackArgs t) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int k = blockIdx.x;
    const TrkReq& rq = t.req[k];
    const int K = t.pcount[k];
    if (K > t.pcap) {
        if (threadIdx.x == 0) t.flags[k] |= kTrkOverflow;
        return;
    }
    int N = 1;
    while (N < K) N <<= 1;
    ulonglong2* list = t.pairs + (int64_t)k * t.pcap;
    const bool in_smem = N <= kSmemPairs;
    ulonglong2* v = in_smem ? reinterpret_cast<ulonglong2*>(smem) : list;
    const ulonglong2 pad = make_ulonglong2(~0ull, ~0ull);
    for (int i = threadIdx.x; i < N; i += blockDim.x) v[i] = i < K ? list[i] : pad;
    __syncthreads();
    bitonic_sort(v, N);
    // bitmaps of taken tracks and detections, and the number of gated pairs per track / detection
    unsigned* tbits = reinterpret_cast<unsigned*>(smem + kSmemPairs * sizeof(ulonglong2));
    unsigned* dbits = tbits + (t.cap + 31) / 32;
    const int nw = (t.cap + 31) / 32 + (t.mcap + 31) / 32;
    int* cnt_t = reinterpret_cast<int*>(tbits + nw);
    int* cnt_d = cnt_t + t.cap;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) tbits[i] = 0u;
    for (int i = threadIdx.x; i < t.cap + t.mcap; i += blockDim.x) cnt_t[i] = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < K; q += blockDim.x) {
        atomicAdd(&cnt_t[(int)(v[q].y >> 32)], 1);
        atomicAdd(&cnt_d[(int)(v[q].y & 0xffffffffu)], 1);
    }
    __syncthreads();
    // A pair whose track and detection are in no other gated pair is taken whatever the order: accept
    // those in parallel.  The greedy outcome of the others depends only on each other (any pair
    // sharing an end with one of them is itself contested), so the sequential scan below runs over
    // the contested pairs alone, in the same sorted order -- the same result as scanning all pairs.
    const int64_t tb = (int64_t)rq.b * t.cap;
    __shared__ int s_tot[32];
    int nc = 0;
    for (int q0 = 0; q0 < K; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        ulonglong2 pr = make_ulonglong2(0ull, 0ull);
        int contested = 0;
        if (q < K) {
            pr = v[q];
            const int i = (int)(pr.y >> 32), j = (int)(pr.y & 0xffffffffu);
            if (cnt_t[i] == 1 && cnt_d[j] == 1) {
                atomicOr(&tbits[i >> 5], 1u << (i & 31));
                atomicOr(&dbits[j >> 5], 1u << (j & 31));
                t.match[tb + i] = j;
            } else {
                contested = 1;
            }
        }
        int tot;
        const int pos = nc + block_scan(contested, s_tot, &tot);  // (block_scan synchronises)
        if (contested) v[pos] = pr;  // stable, in place: pos <= q and this chunk was read above
        nc += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < nc; ++q) {
            const ulonglong2 p = v[q];
            const int i = (int)(p.y >> 32), j = (int)(p.y & 0xffffffffu);
            const unsigned ti = 1u << (i & 31), dj = 1u << (j & 31);
            if ((tbits[i >> 5] & ti) | (dbits[j >> 5] & dj)) continue;
            tbits[i >> 5] |= ti;
            dbits[j >> 5] |= dj;
            t.match[tb + i] = j;
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < rq.m; j += blockDim.x)
        t.used[(int64_t)k * t.mcap + j] = (dbits[j >> 5] >> (j & 31)) & 1u;
}

__global__ void k_trk_update(TrackArgs t) {
    const int k = blockIdx.y;
    const TrkReq& rq = t.req[k];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rq.n || (t.flags[k] & kTrkOverflow)) return;
    const int64_t s = (int64_t)rq.b * t.cap + i;
    int mis = t.missed[s] + 1;
    const int j = t.match[s];
    if (j >= 0) {
        twg_track tr = t.pred[s];
        const double2 z = t.det[rq.det_off + j];
        if (trk_kalman_update(tr.x, tr.P, z.x, z.y, t.r2)) {
            t.pred[s] = tr;
            mis = 0;
        } else {
            atomicOr(&t.flags[k], kTrkSingular);
        }
    }
    t.mis_new[s] = mis;
}

// Block-wide exclusive scan of one flag per thread (1024 threads); returns the prefix, *total.
__device__ __forceinline__ int block_scan(int v, int* sw, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < (int)(blockDim.x >> 5) ? sw[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sw[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int excl = x - v + (w > 0 ? sw[w - 1] : 0);
    *total = sw[(blockDim.x >> 5) - 1];
    __syncthreads();
    return excl;
}

// Positions of the surviving tracks and of the spawned ones (one CTA per request, integer block
// scans only): pos_t[i] (in the match array, free after k_trk_update) and pos_d[j] (in the pair list,
// free after k_trk_assoc), -1 when pruned, matched or beyond the capacity; then k_trk_scatter moves the
// 160-byte tracks with the whole grid.
__global__ void __launch_bounds__(1024) k_trk_compact(TrackArgs t) {
    __shared__ int sw[32];
    const int k = blockIdx.x;
    const TrkReq& rq = t.req[k];
    if (t.flags[k] & kTrkOverflow) return;
    const int64_t tb = (int64_t)rq.b * t.cap;
    int* pos_d = reinterpret_cast<int*>(t.pairs + (int64_t)k * t.pcap);
    const int limit = rq.limit;
    int pos = 0;
    bool trunc = false;
    for (int i0 = 0; i0 < rq.n; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const int keep = (i < rq.n && t.mis_new[tb + i] <= t.prune_after) ? 1 : 0;
        int tot;
        const int p = pos + block_scan(keep, sw, &tot);
        if (i < rq.n) t.match[tb + i] = keep && p < limit ? p : -1;
        trunc |= keep && p >= limit;
        pos += tot;
    }
    for (int j0 = 0; j0 < rq.m; j0 += blockDim.x) {
        const int j = j0 + threadIdx.x;
        const int sp = (j < rq.m && !t.used[(int64_t)k * t.mcap + j]) ? 1 : 0;
        int tot;
        const int p = pos + block_scan(sp, sw, &tot);
        if (j < rq.m) pos_d[j] = sp && p < limit ? p : -1;
        trunc |= sp && p >= limit;
        pos += tot;
    }
    if (__syncthreads_or(trunc) && threadIdx.x == 0) atomicOr(&t.flags[k], kTrkTruncated);
    if (threadIdx.x == 0) t.n_out[k] = min(pos, limit);
}

__global__ void k_trk_scatter(TrackArgs t) {
    const int k = blockIdx.y;
    const TrkReq& rq = t.req[k];
    if (t.flags[k] & kTrkOverflow) return;
    const int64_t tb = (int64_t)rq.b * t.cap;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < rq.n) {
        const int p = t.match[tb + q];
        if (p >= 0) {
            t.trk[tb + p] = t.pred[tb + q];
            t.missed[tb + p] = t.mis_new[tb + q];
        }
    }
    if (q < rq.m) {
        const int p = reinterpret_cast<const int*>(t.pairs + (int64_t)k * t.pcap)[q];
        if (p >= 0) {
            const double2 z = t.det[rq.det_off + q];
            twg_track o;
#pragma unroll
            for (int e = 0; e < 16; ++e) o.P[e] = 0.0;
            o.x[0] = z.x;
            o.x[1] = z.y;
            o.x[2] = 0.0;
            o.x[3] = 0.0;
            o.P[0] = t.var_pos;
            o.P[5] = t.var_pos;
            o.P[10] = t.var_vel;
            o.P[15] = t.var_vel;
            t.trk[tb + p] = o;
            t.missed[tb + p] = 0;
        }
    }
}

cudaError_t launch_track_step(const TrackArgs& t, int nreq, int max_n, int max_m, int* n_launch, cudaStream_t st) {
    static unsigned long long init_mask = 0;
    const size_t smem = kSmemPairs * sizeof(ulonglong2) + ((t.cap + 31) / 32 + (t.mcap + 31) / 32) * sizeof(unsigned) +
                        (size_t)(t.cap + t.mcap) * sizeof(int);
    constexpr size_t kMaxDyn = 227 * 1024 - 1024;  // leaves room for the kernel's static shared memory
    if (smem > kMaxDyn) return cudaErrorInvalidValue;
    if (first_on_device(init_mask))
        cudaFuncSetAttribute(k_trk_assoc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDyn);
    const int nm = std::max(std::max(max_n, max_m), 1);
    k_trk_predict<<<dim3((nm + 127) / 128, nreq), 128, 0, st>>>(t);
    const int tiles = ((max_n + kPairTile - 1) / kPairTile) * ((max_m + kPairTile - 1) / kPairTile);
    k_trk_pairs<<<dim3(std::max(std::min(tiles, 4096), 1), nreq), 256, 0, st>>>(t);
    k_trk_assoc<<<nreq, 1024, smem, st>>>(t);
    k_trk_update<<<dim3((std::max(max_n, 1) + 127) / 128, nreq), 128, 0, st>>>(t);
    k_trk_compact<<<nreq, 1024, 0, st>>>(t);
    k_trk_scatter<<<dim3((nm + 127) / 128, nreq), 128, 0, st>>>(t);
    if (n_launch) *n_launch = 6;
    return cudaGetLastError();
}

void preload_track_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_trk_predict);
    cudaFuncGetAttributes(&a, k_trk_pairs);
    cudaFuncGetAttributes(&a, k_trk_assoc);
    cudaFuncGetAttributes(&a, k_trk_update);
    cudaFuncGetAttributes(&a, k_trk_compact);
    cudaFuncGetAttributes(&a, k_trk_scatter);
    cudaGetLastError();
}

}  // namespace twg
