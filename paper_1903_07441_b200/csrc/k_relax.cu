// k_relax.cu -- rows a4-a6: red-black Laplace relaxation (Eq. 2, realised as
// red-black Gauss-Seidel, C1), the fused max|du| residual (C5) and device-side
// convergence control (C6).
//
// k_rb_tblock<T>: temporally blocked tile kernel.  One warp owns a strip of 128
// columns (4 cells per lane) x hseg output rows.  Input rows arrive through a
// per-warp TMA ring (cp.async.bulk.tensor.3d + mbarrier, OOB zero fill = the
// outside-obstacle boundary C4); the 2T half-sweeps of T sweeps run as a
// register wavefront: when row y lands, half-sweep k (k = 1..2T) updates row
// y - k, so every input cell is read from HBM once per launch and written once
// (8 B per cell per launch), while T lattice updates are performed per cell.
// Halo: 2T rows above/below and round_up(2T, 4) columns left/right are
// recomputed redundantly (SURVEY 0 finding 6).
//
// Bit-exactness with the oracle (oracle/twg_oracle.c orc_relax_f32): each free
// cell becomes 0.25f * ((|E| + |W|) + (|N| + |S|)) -- the same IEEE operation
// sequence (C2; the library is compiled with -fmad=false, no fast-math, no
// FTZ); colours are global (x + row_offset + y) parity; the residual is the
// exact max of fabsf(new - old) over the free cells of the last sweep.
//
// Also here: k_jacobi (Eq. 1, relax mode 1), k_lex (lexicographic Eq. 2, mode 2, a persistent
// tile wavefront), and the convergence control k_check /
// k_fixup.  The launches of a relaxation chain use programmatic dependent launch.
#include <algorithm>

#include "twg_kernels.cuh"

namespace twg {

// Update the cells of parity q (j = q, q + 2 of the lane's float4) of row `c`
// from rows `up` (y - 1) and `dn` (y + 1).  Returns the largest |du| of the
// updated free cells in *dmax when TRACK.
template <int Q, bool TRACK>
__device__ __forceinline__ void half_sweep(float4& c, const float4& up, const float4& dn, float& dmax) {
    if (Q == 0) {
        const float l = __shfl_up_sync(0xffffffffu, c.w, 1);  // cell x - 1 of j = 0 (lane - 1, j = 3)
        const float n0 = 0.25f * ((fabsf(c.y) + fabsf(l)) + (fabsf(up.x) + fabsf(dn.x)));
        const float n2 = 0.25f * ((fabsf(c.w) + fabsf(c.y)) + (fabsf(up.z) + fabsf(dn.z)));
        const bool f0 = is_free(c.x), f2 = is_free(c.z);
        if (TRACK) {
            if (f0) dmax = fmaxf(dmax, fabsf(-n0 - c.x));
            if (f2) dmax = fmaxf(dmax, fabsf(-n2 - c.z));
        }
        c.x = f0 ? -n0 : c.x;
        c.z = f2 ? -n2 : c.z;
    } else {
        const float r = __shfl_down_sync(0xffffffffu, c.x, 1);  // cell x + 1 of j = 3 (lane + 1, j = 0)
        const float n1 = 0.25f * ((fabsf(c.z) + fabsf(c.x)) + (fabsf(up.y) + fabsf(dn.y)));
        const float n3 = 0.25f * ((fabsf(r) + fabsf(c.z)) + (fabsf(up.w) + fabsf(dn.w)));
        const bool f1 = is_free(c.y), f3 = is_free(c.w);
        if (TRACK) {
            if (f1) dmax = fmaxf(dmax, fabsf(-n1 - c.y));
            if (f3) dmax = fmaxf(dmax, fabsf(-n3 - c.w));
        }
        c.y = f1 ? -n1 : c.y;
        c.w = f3 ? -n3 : c.w;
    }
}

// One wavefront step: row i of the strip (global row y = ystart + i) has landed in
// win[S]; run half-sweeps k = 1..2T on rows y - k; store row y - 2T through the running
// output pointer `op` (row i - 4T of the segment; advanced by one pitch per step).
template <int T, int QOFF, bool RESID, int S>
__device__ __forceinline__ void wave_step(float4 (&win)[2 * T + 2], int i, unsigned hs, int rlo, unsigned rn,
                                          bool lane_out, float*& op, int64_t P, float& dmax) {
    constexpr int NW = 2 * T + 2;
    // all half-sweeps of this step update cells of one parity: q = (y + row_offset + 1) & 1
    constexpr int Qp = (S + 1 + QOFF) & 1;
#pragma unroll
    for (int k = 1; k <= 2 * T; ++k) {
        const int c = (S - k + 2 * NW) % NW;
        const int up = (S - k - 1 + 2 * NW) % NW;
        const int dn = (S - k + 1 + 2 * NW) % NW;
        if (RESID && k >= 2 * T - 1) {
            const int r = i - k - 2 * T;  // row index relative to the first output row
            float d = 0.0f;
            half_sweep<Qp, true>(win[c], win[up], win[dn], d);
            if (lane_out && (unsigned)(r - rlo) < rn) dmax = fmaxf(dmax, d);
        } else {
            float d = 0.0f;
            half_sweep<Qp, false>(win[c], win[up], win[dn], d);
        }
    }
    constexpr int so = (S - 2 * T + 2 * NW) % NW;
    if (lane_out && (unsigned)(i - 4 * T) < hs) *reinterpret_cast<float4*>(op) = win[so];
    TWG_CHECK(!(lane_out && (unsigned)(i - 4 * T) < hs) || (unsigned)(i - 4 * T) < hs);
    op += P;
}

// Per-warp streaming state of k_rb_tblock.
struct Strip {
    const float* rows;  // current ring stage: NW rows x 128 floats
    float* op;          // output pointer of the row finalised by the next step
    int64_t P;
    unsigned hs;        // output rows of this segment
    int lane;
    int rlo;            // first row (relative to the first output row) counted in the residual
    unsigned rn;        // number of rows counted in the residual
    bool lane_out;
    float dmax;
    // packed fast path near the goal (GOAL variant): the goal's absolute row, lane, column parity of its
    // pair (0: a, 1: b) and element; ystart = absolute row of step 0
    int ystart, gy, gl, gp, ge;
    int y0, row_lo, row_hi, x, P_cols;  // checked build: the stored rows and columns must lie in the grid
};

// Steps S, S+1, ..., NW-1 of one unrolled block of the row loop.  S is a template parameter so
// that every window slot and every ring offset is a compile-time constant; the block has no
// per-row branch (the row count is padded to a multiple of NW on the host).
template <int T, int QOFF, bool RESID, int S>
__device__ __forceinline__ void block_steps(float4 (&win)[2 * T + 2], int ib, Strip& st) {
    win[S] = reinterpret_cast<const float4*>(st.rows + S * kStripW)[st.lane];
    wave_step<T, QOFF, RESID, S>(win, ib + S, st.hs, st.rlo, st.rn, st.lane_out, st.op, st.P, st.dmax);
    if constexpr (S + 1 < 2 * T + 2) block_steps<T, QOFF, RESID, S + 1>(win, ib, st);
}

// ---------------------------------------------------------------- packed fast path
// Used by every warp whose region holds no positive fixed cell (the goal and any other fixed cell
// with u > 0: RelaxArgs::fixbox); there the only fixed cells are obstacles, u = 0.  The four cells
// of a lane are kept as two parity pairs -- a = columns (4l, 4l+2), b = (4l+1, 4l+3) -- so that the
// two cells of one half-sweep are one register pair and the update runs on the sm_100a packed
// FP32 pipe: (E+W), (N+S), their sum and the scaling are each ONE f32x2 instruction for both cells
// (add.rn.f32x2 / mul.rn.f32x2: the same IEEE round-to-nearest operations as the scalar oracle, no
// FTZ, so the result is bit-identical, C2).  No |.| is needed: in this region every value is <= 0
// (free cells hold -u) or a zero (obstacle), so every sum is -(sum of the magnitudes) exactly
// (round-to-nearest is sign-symmetric) and only the sign of a zero may differ.  The free/fixed
// choice is a per-cell multiplier m (0.25 for a free cell, -0.0 for an obstacle, taken from the
// sign bit when the row lands): u <- m ((E+W) + (N+S)) gives 0.25 (...) for a free cell and a zero
// for an obstacle.  The stored encoding is restored when the row leaves: sign from m, magnitude
// from the value (so a free cell whose value is a +0 is still stored as -0.0).
struct FRow {
    float2 a, b;    // values of the parity pairs
    float2 ma, mb;  // their multipliers
};

__device__ __forceinline__ float2 f2add(float2 x, float2 y) {
    float2 r;
    asm("{\n.reg .b64 X, Y, R;\nmov.b64 X, {%2, %3};\nmov.b64 Y, {%4, %5};\nadd.rn.f32x2 R, X, Y;\n"
        "mov.b64 {%0, %1}, R;\n}" : "=f"(r.x), "=f"(r.y) : "f"(x.x), "f"(x.y), "f"(y.x), "f"(y.y));
    return r;
}
__device__ __forceinline__ float2 f2sub(float2 x, float2 y) {
    float2 r;
    asm("{\n.reg .b64 X, Y, R;\nmov.b64 X, {%2, %3};\nmov.b64 Y, {%4, %5};\nsub.rn.f32x2 R, X, Y;\n"
        "mov.b64 {%0, %1}, R;\n}" : "=f"(r.x), "=f"(r.y) : "f"(x.x), "f"(x.y), "f"(y.x), "f"(y.y));
    return r;
}
__device__ __forceinline__ float2 f2mul(float2 x, float2 y) {
    float2 r;
    asm("{\n.reg .b64 X, Y, R;\nmov.b64 X, {%2, %3};\nmov.b64 Y, {%4, %5};\nmul.rn.f32x2 R, X, Y;\n"
        "mov.b64 {%0, %1}, R;\n}" : "=f"(r.x), "=f"(r.y) : "f"(x.x), "f"(x.y), "f"(y.x), "f"(y.y));
    return r;
}
// 0.25 for a free cell (sign bit set), -0.0 for a fixed one.
__device__ __forceinline__ float mult_of(float c) {
    const int t = __float_as_int(c) >> 31;
    return __int_as_float((t & 0x3E800000) | (~t & (int)0x80000000));
}
// Stored encoding of value v with multiplier m: |v| with the sign bit set iff the cell is free, i.e.
// (v & 0x7fffffff) | (~m & 0x80000000) -- one LOP3 (LUT 0xB1 over v, m, 0x7fffffff).
__device__ __forceinline__ float enc_of(float v, float m) {
    float r;
    asm("lop3.b32 %0, %1, %2, 0x7fffffff, 0xb1;" : "=f"(r) : "f"(v), "f"(m));
    return r;
}

// The goal cell (u = 1, fixed) inside the fast path: held as -1 in registers like a free cell of u = 1
// (its multiplier is the fixed one, so it is stored back as +1.0), and written back to -1 after every
// half-sweep of its row and column parity.
__device__ __forceinline__ void goal_patch(float2& nv, bool hit, int lane, const Strip& st) {
    if (hit && lane == st.gl) {
        if (st.ge) nv.y = -1.0f;
        else nv.x = -1.0f;
    }
}

template <int Q, bool TRACK, bool GOAL>
__device__ __forceinline__ void hs_fast(FRow& c, const FRow& up, const FRow& dn, float& d, bool ghit, const Strip& st) {
    // E + W of the two cells as two scalar FADDs (one operand is the neighbour lane's cell, so the
    // pair would first have to be assembled), (N + S), the sum and the scaling packed
    if (Q == 0) {  // cells 4l, 4l+2: E = (4l+1, 4l+3) = b, W = (4l-1, 4l+1)
        const float l = __shfl_up_sync(0xffffffffu, c.b.y, 1);
        const float2 ew = make_float2(c.b.x + l, c.b.y + c.b.x);
        float2 nv = f2mul(f2add(ew, f2add(up.a, dn.a)), c.ma);
        if (GOAL) goal_patch(nv, ghit, st.lane, st);
        if (TRACK) {
            const float2 dd = f2sub(nv, c.a);
            d = fmaxf(fabsf(dd.x), fabsf(dd.y));
        }
        c.a = nv;
    } else {  // cells 4l+1, 4l+3: E = (4l+2, 4l+4), W = (4l, 4l+2) = a
        const float r = __shfl_down_sync(0xffffffffu, c.a.x, 1);
        const float2 ew = make_float2(c.a.y + c.a.x, r + c.a.y);
        float2 nv = f2mul(f2add(ew, f2add(up.b, dn.b)), c.mb);
        if (GOAL) goal_patch(nv, ghit, st.lane, st);
        if (TRACK) {
            const float2 dd = f2sub(nv, c.b);
            d = fmaxf(fabsf(dd.x), fabsf(dd.y));
        }
        c.b = nv;
    }
}

// Half-sweep k of step S (row i - k of the strip, i = ib + S): the packed update plus, on the
// residual sweeps, |du| of the owned rows.
// `upr`: the row above (slot of row i - K - 1), passed separately because for K = 2T that slot may
// already hold the next row (the interleaved order below loads row S + 1 early).
// FIRST: the segment's first block, whose half-sweep k of step S only touches rows above every row
// the stored rows depend on when 2k > S (those rows are never read by a needed update) -- skipped.
template <int T, int QOFF, bool RESID, bool GOAL, bool FIRST, int S, int K>
__device__ __forceinline__ void fast_hs(FRow (&win)[2 * T + 2], const FRow& upr, int i, const Strip& st,
                                        float& dmax) {
    if constexpr (FIRST && 2 * K > S) return;
    constexpr int NW = 2 * T + 2;
    constexpr int Qp = (S + 1 + QOFF) & 1;
    constexpr int c = (S - K + 2 * NW) % NW, dn = (S - K + 1 + 2 * NW) % NW;
    const bool ghit = GOAL && st.gp == Qp && st.ystart + i - K == st.gy;
    if (RESID && K >= 2 * T - 1) {
        float d = 0.0f;
        hs_fast<Qp, true, GOAL>(win[c], upr, win[dn], d, ghit, st);
        const int r = i - K - 2 * T;
        if (st.lane_out && (unsigned)(r - st.rlo) < st.rn) dmax = fmaxf(dmax, d);
    } else {
        float d = 0.0f;
        hs_fast<Qp, false, GOAL>(win[c], upr, win[dn], d, ghit, st);
    }
}
template <int T, int S, int K>
__device__ __forceinline__ const FRow& up_of(FRow (&win)[2 * T + 2]) {
    return win[(S - K - 1 + 2 * (2 * T + 2)) % (2 * T + 2)];
}

template <int T, bool GOAL, int S>
__device__ __forceinline__ void fast_load(FRow (&win)[2 * T + 2], const Strip& st) {
    const float4 q = reinterpret_cast<const float4*>(st.rows + S * kStripW)[st.lane];
    if (GOAL) {  // every value non-positive: the goal's +1.0 becomes -1 (obstacles -0, free cells unchanged)
        const float4 n = make_float4(-fabsf(q.x), -fabsf(q.y), -fabsf(q.z), -fabsf(q.w));
        win[S].a = make_float2(n.x, n.z);
        win[S].b = make_float2(n.y, n.w);
    } else {
        win[S].a = make_float2(q.x, q.z);
        win[S].b = make_float2(q.y, q.w);
    }
    win[S].ma = make_float2(mult_of(q.x), mult_of(q.z));
    win[S].mb = make_float2(mult_of(q.y), mult_of(q.w));
}

// Row i - 2T is final after step S: store it (stored encoding, predicated store -- no divergent branch,
// so the following shuffles need no reconvergence).
template <int T, int S>
__device__ __forceinline__ void fast_store(FRow (&win)[2 * T + 2], int i, Strip& st) {
    constexpr int NW = 2 * T + 2;
    constexpr int so = (S - 2 * T + 2 * NW) % NW;
    const FRow& w = win[so];
    const float4 o =
        make_float4(enc_of(w.a.x, w.ma.x), enc_of(w.b.x, w.mb.x), enc_of(w.a.y, w.ma.y), enc_of(w.b.y, w.mb.y));
    TWG_CHECK(!(st.lane_out && (unsigned)(i - 4 * T) < st.hs) ||
              (st.y0 + i - 4 * T >= st.row_lo && st.y0 + i - 4 * T < st.row_hi && st.x + 3 < st.P_cols));
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n@p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n}" ::"l"(st.op),
                 "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w), "r"((st.lane_out && (unsigned)(i - 4 * T) < st.hs) ? 1 : 0));
    st.op += st.P;
}

// Steps S and S + 1 with their half-sweeps interleaved along the anti-diagonals of the wavefront:
// (S, k) needs (S, k - 1), (S - 1, k - 1) and (S - 2, k - 1) only, so (S, k) and (S + 1, k - 1) are
// independent and issue back to back -- two dependency chains per warp instead of one.
template <int T, int QOFF, bool RESID, bool GOAL, bool FIRST, int S, int K>
__device__ __forceinline__ void fast_pair_hs(FRow (&win)[2 * T + 2], const FRow& last_up, int ib, const Strip& st,
                                             float& dmax) {
    if constexpr (K <= 2 * T) {
        if constexpr (K == 2 * T) fast_hs<T, QOFF, RESID, GOAL, FIRST, S, K>(win, last_up, ib + S, st, dmax);
        else fast_hs<T, QOFF, RESID, GOAL, FIRST, S, K>(win, up_of<T, S, K>(win), ib + S, st, dmax);
        fast_hs<T, QOFF, RESID, GOAL, FIRST, S + 1, K - 1>(win, up_of<T, S + 1, K - 1>(win), ib + S + 1, st, dmax);
        fast_pair_hs<T, QOFF, RESID, GOAL, FIRST, S, K + 1>(win, last_up, ib, st, dmax);
    }
}

template <int T, int QOFF, bool RESID, bool GOAL, bool FIRST, int S>
__device__ __forceinline__ void block_steps_fast(FRow (&win)[2 * T + 2], int ib, Strip& st) {
    constexpr int NW = 2 * T + 2;
    float dmax = st.dmax;
    fast_load<T, GOAL, S>(win, st);
    fast_hs<T, QOFF, RESID, GOAL, FIRST, S, 1>(win, up_of<T, S, 1>(win), ib + S, st, dmax);
    // row S + 1 lands in the slot of row S - 2T - 1, which (S, 2T) still reads as its upper neighbour
    const FRow last_up = win[(S + 1) % NW];
    fast_load<T, GOAL, S + 1>(win, st);
    fast_pair_hs<T, QOFF, RESID, GOAL, FIRST, S, 2>(win, last_up, ib, st, dmax);
    fast_store<T, S>(win, ib + S, st);
    fast_hs<T, QOFF, RESID, GOAL, FIRST, S + 1, 2 * T>(win, up_of<T, S + 1, 2 * T>(win), ib + S + 1, st, dmax);
    fast_store<T, S + 1>(win, ib + S + 1, st);
    st.dmax = dmax;
    if constexpr (S + 2 < 2 * T + 2) block_steps_fast<T, QOFF, RESID, GOAL, FIRST, S + 2>(win, ib, st);
}

// The fast path's row loop.  has_goal: the goal cell lies in the warp's region; it is loaded at step
// i0 = gy - ystart, updated at steps i0 + 1 .. i0 + 2T and read by its neighbours until step
// i0 + 2T + 1, so only the (at most two) blocks holding steps i0 .. i0 + 2T run the GOAL variant (load
// as -|u|, write the goal back after its half-sweeps); outside them the goal row is either not yet
// loaded or only read (its -1 is kept in the register).
template <int T, int QOFF, bool RESID>
__device__ __forceinline__ void fast_rows(float* ring, uint64_t* bars, const CUtensorMap* tmap, int xb, int b, int nblk,
                                          bool has_goal, Strip& st) {
    constexpr int NW = 2 * T + 2;
    constexpr int STAGE_F = NW * kStripW;
    FRow win[NW];
#pragma unroll
    for (int s = 0; s < NW; ++s) win[s] = FRow{make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                               make_float2(0.f, 0.f)};
    const int i0 = st.gy - st.ystart;
    for (int blk = 0; blk < nblk; ++blk) {
        const int sg = blk % kStages;
        mbar_wait(&bars[sg], (blk / kStages) & 1);
        st.rows = ring + sg * STAGE_F;
        const bool gblk = has_goal && blk * NW <= i0 + 2 * T && blk * NW + NW - 1 >= i0;
        if (blk == 0) {
            if (gblk) block_steps_fast<T, QOFF, RESID, true, true, 0>(win, 0, st);
            else block_steps_fast<T, QOFF, RESID, false, true, 0>(win, 0, st);
        } else {
            if (gblk) block_steps_fast<T, QOFF, RESID, true, false, 0>(win, blk * NW, st);
            else block_steps_fast<T, QOFF, RESID, false, false, 0>(win, blk * NW, st);
        }
        if (blk + kStages < nblk) {
            __syncwarp();
            if (st.lane == 0) {
                mbar_expect_tx(&bars[sg], STAGE_F * 4);
                tma_load_3d(ring + sg * STAGE_F, tmap, xb, st.ystart + (blk + kStages) * NW, b, &bars[sg]);
            }
        }
    }
}

template <int T, int QOFF, bool RESID>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_rb_tblock(const __grid_constant__ CUtensorMap tmap0, const __grid_constant__ CUtensorMap tmap1, RelaxArgs a) {
    constexpr int NW = 2 * T + 2;          // rows per TMA box = rows per unrolled block
    constexpr int HX = halo_cols(T);
    constexpr int WOUT = out_cols(T);
    constexpr int STAGE_F = NW * kStripW;  // floats per ring stage
    pdl_wait();
    const int b = blockIdx.y;
    if (a.done != nullptr && a.done[b]) return;  // scenario converged: whole CTA exits
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nseg = a.seg_end - a.seg_begin;
    const int task = blockIdx.x * kWarpsPerCta + warp;
    if (task >= a.n_strips * nseg) return;  // warp-local from here on (no CTA barriers)
    const int strip = task % a.n_strips;
    const int seg = a.seg_begin + task / a.n_strips;
    const int src = a.cur[b] ^ a.lp;  // buffer read by this launch; the other one is written
    const CUtensorMap* tmap = src ? &tmap1 : &tmap0;

    const int xb = strip * WOUT - HX;  // first (halo) column of the strip, even
    const int y0 = a.row_lo + seg * a.hseg;  // first output row (its parity is folded into QOFF)
    Strip st;
    const int hs = min(a.hseg, a.row_hi - y0);
    st.hs = (unsigned)hs;
    st.rlo = max(0, a.res_r0 - y0);
    st.rn = (unsigned)max(0, min(hs, a.res_r1 - y0) - st.rlo);
    const int ystart = y0 - 2 * T;
    const int nblk = (hs + 4 * T + NW - 1) / NW;  // rows ystart .. ystart + nblk*NW - 1
    st.lane = lane;
    st.P = a.P;
    st.y0 = y0;
    st.row_lo = a.row_lo;
    st.row_hi = a.row_hi;
    st.P_cols = (int)a.P;

    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem) + warp * (kStages * STAGE_F);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWarpsPerCta * kStages * STAGE_F * 4) + warp * kStages;

    if (lane == 0) {
        prefetch_tmap(tmap);
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        for (int c = 0; c < kStages && c < nblk; ++c) {
            mbar_expect_tx(&bars[c], STAGE_F * 4);
            tma_load_3d(ring + c * STAGE_F, tmap, xb, ystart + c * NW, b, &bars[c]);
        }
    }
    __syncwarp();

    const int x = xb + 4 * lane;
    st.lane_out = lane >= HX / 4 && lane < 32 - HX / 4 && x < a.W;
    st.x = x;
    TWG_CHECK(y0 >= a.row_lo && y0 < a.row_hi && hs > 0);
    // row i - 4T of the segment is finalised at step i: start 4T rows above the first output row
    st.op = (src ? a.u0 : a.u1) + (int64_t)b * a.sstride + (int64_t)(y0 - 4 * T) * a.P + x;
    st.dmax = 0.0f;
    // the packed fast path unless the warp's region [xb, xb + 128) x [ystart, ystart + nblk NW) holds a
    // positive fixed cell (goal box, imported-field box) -- warp-uniform
    // the goal (box 0, a single cell) takes the fast path's GOAL variant; any other positive fixed cell
    // (box 1: an imported field) the scalar path
    bool slow = a.force_slow == 1, goal = false;
    st.ystart = ystart;
    if (a.fixbox != nullptr && a.force_slow != 2) {
        const int yend = ystart + nblk * NW - 1;
        auto hits = [&](const int4 fb) {  // (x0, x1, y0, y1), empty when x0 > x1
            return fb.x <= fb.y && fb.x <= xb + kStripW - 1 && fb.y >= xb && fb.z <= yend && fb.w >= ystart;
        };
        const int4 g = a.fixbox[2 * b];
        slow = slow || hits(a.fixbox[2 * b + 1]) || (hits(g) && (g.x != g.y || g.z != g.w));
        goal = !slow && hits(g);
        st.gy = g.z;
        st.gl = (g.x - xb) >> 2;
        st.gp = (g.x - xb) & 1;
        st.ge = ((g.x - xb) >> 1) & 1;
    }
    if (slow) {
        float4 win[NW];
#pragma unroll
        for (int s = 0; s < NW; ++s) win[s] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int blk = 0; blk < nblk; ++blk) {
            const int sg = blk % kStages;
            mbar_wait(&bars[sg], (blk / kStages) & 1);
            st.rows = ring + sg * STAGE_F;
            block_steps<T, QOFF, RESID, 0>(win, blk * NW, st);
            if (blk + kStages < nblk) {
                __syncwarp();  // every lane has consumed stage sg (its values are in registers)
                if (lane == 0) {
                    mbar_expect_tx(&bars[sg], STAGE_F * 4);
                    tma_load_3d(ring + sg * STAGE_F, tmap, xb, ystart + (blk + kStages) * NW, b, &bars[sg]);
                }
            }
        }
    } else {
        fast_rows<T, QOFF, RESID>(ring, bars, tmap, xb, b, nblk, goal, st);
    }

    pdl_trigger();
    if (RESID) {
        const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(st.dmax));
        if (lane == 0 && m != 0u) atomicMax(&a.res[b], m);
    }
}

// ---------------------------------------------------------------- small grids: one CTA, whole solve
// Grids whose field fits in shared memory (W H <= kSmallCells, e.g. C1's 64^2) are relaxed by one CTA
// per scenario in a single launch: the field is staged in shared memory, every half-sweep is a block-
// wide pass over one colour (in place: cells of one colour never neighbour each other) separated by
// barriers, and the residual (max |du| of the sweep's free cells, C5) and the stop rule (C6) are
// evaluated on the device after every check sweep -- the same operations as the tile kernel and the
// oracle, without one launch (plus one k_check) per chunk.  The result is written back in place.
constexpr int kSmallCells = 40960;  // 160 KiB of shared memory
constexpr int kSmallThreads = 1024;  // 32 warps (measured: 512 / 256 threads 7 % / 64 % slower on C1)

__global__ void __launch_bounds__(kSmallThreads) k_rb_small(RelaxArgs a, int max_sweeps, int check_every, float tol,
                                                            int qoff, int* __restrict__ sweeps_out,
                                                            float* __restrict__ res_out) {
    extern __shared__ float sf[];  // [H][W]
    __shared__ unsigned s_red[kSmallThreads / 32];
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x;
    if (a.done[b]) return;
    const int W = a.W, H = a.H, n = W * H;
    float* g = (a.cur[b] ? a.u1 : a.u0) + (int64_t)b * a.sstride;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NWARP = kSmallThreads / 32;
    for (int y = wid; y < H; y += NWARP)
        for (int x = lane; x < W; x += 32) sf[y * W + x] = g[(int64_t)y * a.P + x];
    __syncthreads();
    float res = 0.0f;
    int s = 0;
    for (s = 1; s <= max_sweeps; ++s) {
        const bool check = (s % check_every == 0) || s == max_sweeps;
        float dmax = 0.0f;
#pragma unroll 1
        for (int color = 0; color < 2; ++color) {
            // rows y and y + NWARP together (same colour offset: NWARP is even), every load of both issued
            // before any store -- cells of one colour never neighbour each other, so the stores cannot
            // feed the loads of the same pass
            for (int y = wid; y < H; y += 2 * NWARP) {
                // cells of this colour in row y: (x + row_offset + y) & 1 == color
                const int x0 = (color + qoff + y) & 1;
                const int y2 = y + NWARP;
                const bool has2 = y2 < H;
                const bool cnt1 = check && y >= a.res_r0 && y < a.res_r1;
                const bool cnt2 = check && has2 && y2 >= a.res_r0 && y2 < a.res_r1;
                float* row1 = sf + y * W;
                float* row2 = sf + (has2 ? y2 : y) * W;
                for (int x = x0 + 2 * lane; x < W; x += 64) {
                    const float c1 = row1[x];
                    const float e1 = x + 1 < W ? fabsf(row1[x + 1]) : 0.0f;
                    const float w1 = x > 0 ? fabsf(row1[x - 1]) : 0.0f;
                    const float n1 = y > 0 ? fabsf(row1[x - W]) : 0.0f;
                    const float s1 = y + 1 < H ? fabsf(row1[x + W]) : 0.0f;
                    const float c2 = row2[x];
                    const float e2 = x + 1 < W ? fabsf(row2[x + 1]) : 0.0f;
                    const float w2 = x > 0 ? fabsf(row2[x - 1]) : 0.0f;
                    const float n2 = has2 ? fabsf(row2[x - W]) : 0.0f;  // y2 >= NWARP > 0
                    const float s2 = y2 + 1 < H ? fabsf(row2[x + W]) : 0.0f;
                    const float nv1 = 0.25f * ((e1 + w1) + (n1 + s1));
                    const float nv2 = 0.25f * ((e2 + w2) + (n2 + s2));
                    if (is_free(c1)) {
                        if (cnt1) dmax = fmaxf(dmax, fabsf(-nv1 - c1));
                        row1[x] = -nv1;
                    }
                    if (has2 && is_free(c2)) {
                        if (cnt2) dmax = fmaxf(dmax, fabsf(-nv2 - c2));
                        row2[x] = -nv2;
                    }
                }
            }
            __syncthreads();
        }
        if (check) {
            const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(dmax));
            if (lane == 0) s_red[wid] = m;
            __syncthreads();
            // every warp reduces the warp maxima itself (one shared load per lane and a warp max), so the
            // block needs no second round trip through shared memory
            const unsigned mm = __reduce_max_sync(0xffffffffu, lane < NWARP ? s_red[lane] : 0u);
            res = __uint_as_float(mm);
            __syncthreads();  // s_red is rewritten at the next check
            if ((s % check_every == 0 && res < tol) || s == max_sweeps) break;
        }
    }
    if (s > max_sweeps) s = max_sweeps;
    (void)n;
    for (int y = wid; y < H; y += NWARP)
        for (int x = lane; x < W; x += 32) g[(int64_t)y * a.P + x] = sf[y * W + x];
    if (threadIdx.x == 0) {
        sweeps_out[b] = s;
        res_out[b] = res;
    }
}

bool small_grid(int W, int H) { return (int64_t)W * H <= kSmallCells; }

cudaError_t launch_rb_small(const RelaxArgs& a, int B, int max_sweeps, int check_every, float tol, int qoff,
                            int* sweeps_out, float* res_out, cudaStream_t st) {
    const size_t smem = (size_t)a.W * a.H * sizeof(float);
    static unsigned long long attr_mask = 0;
    if (first_on_device(attr_mask))
        cudaFuncSetAttribute(k_rb_small, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallCells * (int)sizeof(float));
    cudaError_t e = launch_pdl(k_rb_small, dim3(B), dim3(kSmallThreads), smem, st, a, max_sweeps, check_every, tol, qoff,
                               sweeps_out, res_out);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Jacobi
// Eq. 1: every free cell from the previous iterate, u <- 0.25 ((E + W) + (N + S)), read
// from buffer cur[b] ^ lp and written to the other one (fixed cells copied through).  One sweep per
// launch; HBM-bound (4 B read + 4 B written per cell).  A warp owns a 128-column strip (float4 per
// lane) and marches down kJacRows rows keeping rows y - 1, y, y + 1 in registers; the E/W neighbours
// come from the adjacent lanes by shuffle, the strip-edge ones from two scalar loads.
constexpr int kJacRows = 16, kJacWarps = 4;

__device__ __forceinline__ float jac_cell(float c, float e, float w, float n, float s, float& dmax, bool count) {
    if (!is_free(c)) return c;
    const float nv = 0.25f * ((fabsf(e) + fabsf(w)) + (fabsf(n) + fabsf(s)));
    if (count) dmax = fmaxf(dmax, fabsf(-nv - c));
    return -nv;
}

__global__ void __launch_bounds__(kJacWarps * 32) k_jacobi(RelaxArgs a, int resid) {
    pdl_wait();
    const int b = blockIdx.z;
    if (a.done[b]) return;
    const int lane = threadIdx.x & 31;
    const int x0 = blockIdx.x * kStripW;
    const int x = x0 + 4 * lane;
    const int y0 = (blockIdx.y * kJacWarps + (threadIdx.x >> 5)) * kJacRows;
    if (y0 >= a.H) return;  // warp-uniform
    const int src_i = a.cur[b] ^ a.lp;
    const float* __restrict__ src = (src_i ? a.u1 : a.u0) + (int64_t)b * a.sstride;
    float* __restrict__ dst = (src_i ? a.u0 : a.u1) + (int64_t)b * a.sstride;
    const bool in = x < a.P;  // P is a multiple of 32: a float4 is wholly inside or outside the row
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    auto ld4 = [&](int y) -> float4 {
        return (in && y >= 0 && y < a.H) ? __ldg(reinterpret_cast<const float4*>(src + (int64_t)y * a.P + x)) : zero;
    };
    float4 up = ld4(y0 - 1), c = ld4(y0);
    const int y1 = min(y0 + kJacRows, a.H);
    float dmax = 0.0f;
    for (int y = y0; y < y1; ++y) {
        const float4 dn = ld4(y + 1);
        float wv = __shfl_up_sync(0xffffffffu, c.w, 1);
        float ev = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (lane == 0) wv = x0 > 0 ? __ldg(src + (int64_t)y * a.P + x0 - 1) : 0.0f;
        if (lane == 31) ev = x0 + kStripW < a.P ? __ldg(src + (int64_t)y * a.P + x0 + kStripW) : 0.0f;
        if (in) {
            const bool count = resid && y >= a.res_r0 && y < a.res_r1;
            float4 o;
            o.x = jac_cell(c.x, c.y, wv, up.x, dn.x, dmax, count);
            o.y = jac_cell(c.y, c.z, c.x, up.y, dn.y, dmax, count);
            o.z = jac_cell(c.z, c.w, c.y, up.z, dn.z, dmax, count);
            o.w = jac_cell(c.w, ev, c.z, up.w, dn.w, dmax, count);
            *reinterpret_cast<float4*>(dst + (int64_t)y * a.P + x) = o;
        }
        up = c;
        c = dn;
    }
    pdl_trigger();
    if (resid) {
        const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(dmax));
        if (lane == 0 && m != 0u) atomicMax(&a.res[b], m);
    }
}

cudaError_t launch_jacobi(const RelaxArgs& a, int B, bool resid, cudaStream_t st) {
    dim3 grid((unsigned)((a.P + kStripW - 1) / kStripW), (a.H + kJacWarps * kJacRows - 1) / (kJacWarps * kJacRows), B);
    cudaError_t e = launch_pdl(k_jacobi, grid, dim3(kJacWarps * 32), 0, st, a, resid ? 1 : 0);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- lexicographic Gauss-Seidel (f3)
// Eq. 2 literally: in each sweep the cells are updated in row-major order in place, so a
// cell sees this sweep's W and N neighbours and the previous sweep's E and S.  The grid is cut into
// 32 x 32 tiles; tile (i, j) of sweep s may run once tiles (i - 1, j) and (i, j - 1) have finished
// sweep s and tiles (i + 1, j), (i, j + 1) and (i, j) itself have finished sweep s - 1 (their old
// values are what it reads).  A persistent grid of warps takes (sweep, tile, scenario) tasks from a
// global counter in wavefront-time order (tile diagonal + 2 sweep, so consecutive sweeps overlap and
// every dependency is listed first), waits on per-tile sweep counters
// (acquire loads; never on a task no running warp holds, so it cannot deadlock), stages the tile
// plus a 1-cell halo in shared memory (L2 loads, bypassing L1), runs the 63 anti-diagonals of the
// tile with one lane per row -- the same row-major order inside the tile -- and writes it back
// before publishing its counter (release).  Several sweeps are in flight at once (a wavefront of
// tiles per sweep, consecutive sweeps two tile diagonals apart).
constexpr int kLexT = 32, kLexWarps = 4, kLexPitch = kLexT + 2;

__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kLexWarps * 32) k_lex(LexArgs a) {
    __shared__ float tile[kLexWarps][kLexPitch][kLexPitch + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float (*T)[kLexPitch + 1] = tile[warp];
    const unsigned total = (unsigned)a.ntasks * (unsigned)a.B;
    constexpr int kStage = (kLexPitch * kLexPitch + 31) / 32;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(a.task, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= total) break;
        const int b = (int)(t % (unsigned)a.B);
        if (a.done[b]) continue;
        const int2 tk = a.tasks[t / (unsigned)a.B];  // (i | s << 16, j)
        const int ti = tk.x & 0xffff, s = tk.x >> 16, tj = tk.y;
        const int tid = tj * a.TX + ti;
        int* td = a.tdone + (int64_t)b * a.ntiles;
        const int need = a.base + s;  // sweeps this tile has finished before this task
        // lanes 0..4 poll the five counters together (one L2 round trip per poll), then a fence
        // orders the staging loads after what was observed
        const int* dp = td + tid;
        int dv = need;
        bool has = lane == 0;
        if (lane == 1) { has = ti > 0; dp = td + tid - 1; dv = need + 1; }
        if (lane == 2) { has = tj > 0; dp = td + tid - a.TX; dv = need + 1; }
        if (lane == 3) { has = ti + 1 < a.TX; dp = td + tid + 1; }
        if (lane == 4) { has = tj + 1 < a.TY; dp = td + tid + a.TX; }
        unsigned ns = 32;  // exponential back-off keeps the polling of waiting warps off the L2
        while (!__all_sync(0xffffffffu, !has || ld_relaxed(dp) >= dv)) {
            __nanosleep(ns);
            ns = min(ns * 2u, 512u);
        }
        __threadfence();
        float* f = (a.cur[b] ? a.u1 : a.u0) + (int64_t)b * a.sstride;
        const int x0 = ti * kLexT, y0 = tj * kLexT;
        // stage rows y0 - 1 .. y0 + 32, columns x0 - 1 .. x0 + 32 (outside the grid: obstacle 0):
        // all loads first (L2, bypassing the non-coherent L1), then the shared-memory stores
        float v[kStage];
#pragma unroll
        for (int k = 0; k < kStage; ++k) {
            const int q = lane + 32 * k;
            const int rr = q / kLexPitch, cc = q - rr * kLexPitch;
            const int gy = y0 - 1 + rr, gx = x0 - 1 + cc;
            v[k] = (q < kLexPitch * kLexPitch && gy >= 0 && gy < a.H && gx >= 0 && gx < a.W)
                       ? __ldcg(f + (int64_t)gy * a.P + gx)
                       : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < kStage; ++k) {
            const int q = lane + 32 * k;
            const int rr = q / kLexPitch, cc = q - rr * kLexPitch;
            if (q < kLexPitch * kLexPitch) T[rr][cc] = v[k];
        }
        __syncwarp();
        const bool last = s + 1 == a.sweeps;
        const int gy = y0 + lane;
        const bool row_in = gy < a.H;
        const bool count = last && a.res != nullptr && gy >= a.res_r0 && gy < a.res_r1;
        float dmax = 0.0f;
        for (int step = 0; step < 2 * kLexT - 1; ++step) {
            const int x = step - lane;
            if (row_in && x >= 0 && x < kLexT && x0 + x < a.W) {
                const float c = T[lane + 1][x + 1];
                if (is_free(c)) {
                    const float nv = 0.25f * ((fabsf(T[lane + 1][x + 2]) + fabsf(T[lane + 1][x])) +
                                              (fabsf(T[lane][x + 1]) + fabsf(T[lane + 2][x + 1])));
                    if (count) dmax = fmaxf(dmax, fabsf(-nv - c));
                    T[lane + 1][x + 1] = -nv;
                }
            }
            __syncwarp();
        }
        for (int rr = 0; rr < kLexT; ++rr) {
            const int yy = y0 + rr, xx = x0 + lane;
            if (yy < a.H && xx < a.W) f[(int64_t)yy * a.P + xx] = T[rr + 1][lane + 1];
        }
        if (last) {
            const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(dmax));
            if (lane == 0 && m != 0u && a.res != nullptr) atomicMax(&a.res[b], m);
        }
        __threadfence();  // every lane's tile stores before the counter
        __syncwarp();
        if (lane == 0) st_relaxed(td + tid, need + 1);
    }
}

cudaError_t launch_lex(const LexArgs& a, int n_sm, cudaStream_t st) {
    // 8 warps per SM: the wavefront exposes a few thousand ready tasks at most, and every extra
    // waiting warp only adds polling
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lex, kLexWarps * 32, 0);
    const int blocks = std::max(1, n_sm * std::min(std::max(per_sm, 1), 2));
    k_lex<<<blocks, kLexWarps * 32, 0, st>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- convergence control (a6)
// Reset the per-call control of a relaxation in which every scenario takes part and the buffer
// indices are already on the device: done 0, sweeps 0, where -1, residual 0.
__global__ void k_relax_init(int B, int* __restrict__ done, int* __restrict__ sweeps, int* __restrict__ where,
                             unsigned* __restrict__ res_bits, float* __restrict__ res) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    done[b] = 0;
    sweeps[b] = 0;
    where[b] = -1;
    res_bits[b] = 0u;
    res[b] = 0.0f;
}

cudaError_t launch_relax_init(int* done, int* sweeps, int* where, unsigned* res_bits, float* res, int B, cudaStream_t st) {
    cudaError_t e = launch_pdl(k_relax_init, dim3((B + 127) / 128), dim3(128), 0, st, B, done, sweeps, where, res_bits, res);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Residual max over the slabs of a local row-slab group: every slab's residual bits
// become the group maximum (non-negative floats order as their bit patterns).
struct GroupRes {
    unsigned* p[kMaxLocalSlabs];
};
__global__ void k_res_group_max(GroupRes g, int n, int B) {
    pdl_enter();
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        unsigned m = 0u;
        for (int r = 0; r < n; ++r) m = max(m, g.p[r][b]);
        for (int r = 0; r < n; ++r) g.p[r][b] = m;
    }
}

cudaError_t launch_res_group_max(unsigned* const* ptrs, int n, int B, cudaStream_t st) {
    GroupRes g;
    for (int r = 0; r < kMaxLocalSlabs; ++r) g.p[r] = r < n ? ptrs[r] : nullptr;
    k_res_group_max<<<1, 256, 0, st>>>(g, n, B);
    return cudaGetLastError();
}

// After a chunk of `chunk` sweeps whose last launch accumulated the residual:
// sweeps += chunk; stop when (sweeps % check_every == 0 && res < tol) or
// sweeps == max_sweeps (C6).  `where` records which ping-pong buffer
// holds the scenario's field at the time it finished.
__global__ void k_check(int B, int* __restrict__ done, int* __restrict__ sweeps, unsigned* __restrict__ res_bits,
                        float* __restrict__ res_final, int* __restrict__ where, int chunk, int check_every,
                        int max_sweeps, float tol, const int* __restrict__ cur, int lp) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B || done[b]) return;
    const int s = sweeps[b] + chunk;
    sweeps[b] = s;
    const float r = __uint_as_float(res_bits[b]);
    res_final[b] = r;
    res_bits[b] = 0u;
    where[b] = cur[b] ^ lp;
    if ((s % check_every == 0 && r < tol) || s >= max_sweeps) done[b] = 1;
}

// Scenarios that stopped early hold their field in buffer where[b]; move it to the buffer
// cur[b] ^ lp that the host assumes after the call.
__global__ void k_fixup(float* __restrict__ u0, float* __restrict__ u1, int64_t sstride, const int* __restrict__ where,
                        const int* __restrict__ cur, int lp) {
    const int b = blockIdx.y;
    const int tgt = cur[b] ^ lp;
    if (where[b] < 0 || where[b] == tgt) return;  // not relaxed in this call, or already in place
    const float4* src = reinterpret_cast<const float4*>((tgt ? u0 : u1) + (int64_t)b * sstride);
    float4* dst = reinterpret_cast<float4*>((tgt ? u1 : u0) + (int64_t)b * sstride);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < sstride / 4; q += (int64_t)gridDim.x * blockDim.x)
        dst[q] = src[q];
}

// ---------------------------------------------------------------- host launchers
template <int T, int QOFF, bool RESID>
static cudaError_t launch_T(const CUtensorMap& m0, const CUtensorMap& m1, const RelaxArgs& a, int B, cudaStream_t st) {
    const int nseg = a.seg_end - a.seg_begin;
    const int tasks = a.n_strips * nseg;
    dim3 grid((tasks + kWarpsPerCta - 1) / kWarpsPerCta, B);
    const size_t smem = (size_t)kWarpsPerCta * kStages * (2 * T + 2) * kStripW * 4 + kWarpsPerCta * kStages * sizeof(uint64_t);
    static unsigned long long attr_mask = 0;
    if (first_on_device(attr_mask)) {
        cudaFuncSetAttribute(k_rb_tblock<T, QOFF, RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    cudaError_t e = launch_pdl(k_rb_tblock<T, QOFF, RESID>, grid, dim3(kWarpsPerCta * 32), smem, st, m0, m1, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// CTAs of k_rb_tblock<T> resident per SM (registers, shared memory), per process.
template <int T>
static int ctas_per_sm_T() {
    static int n = -1;
    if (n < 0) {
        const size_t smem = (size_t)kWarpsPerCta * kStages * (2 * T + 2) * kStripW * 4 + kWarpsPerCta * kStages * sizeof(uint64_t);
        cudaFuncSetAttribute(k_rb_tblock<T, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int k = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, k_rb_tblock<T, 0, false>, kWarpsPerCta * 32, smem) !=
            cudaSuccess) {
            cudaGetLastError();
            k = 1;
        }
        n = std::max(k, 1);
    }
    return n;
}

int rb_tblock_ctas_per_sm(int T) {
    switch (T) {
        case 1: return ctas_per_sm_T<1>();
        case 2: return ctas_per_sm_T<2>();
        case 3: return ctas_per_sm_T<3>();
        case 4: return ctas_per_sm_T<4>();
        case 5: return ctas_per_sm_T<5>();
        case 6: return ctas_per_sm_T<6>();
        case 7: return ctas_per_sm_T<7>();
        default: return ctas_per_sm_T<8>();
    }
}

template <int T>
static cudaError_t launch_T3(const CUtensorMap& m0, const CUtensorMap& m1, const RelaxArgs& a, int B, int qoff, bool resid,
                             cudaStream_t st) {
    if (qoff) return resid ? launch_T<T, 1, true>(m0, m1, a, B, st) : launch_T<T, 1, false>(m0, m1, a, B, st);
    return resid ? launch_T<T, 0, true>(m0, m1, a, B, st) : launch_T<T, 0, false>(m0, m1, a, B, st);
}

cudaError_t launch_rb_tblock(int T, const CUtensorMap& m0, const CUtensorMap& m1, const RelaxArgs& a, int B, int qoff,
                             bool resid, cudaStream_t st) {
    switch (T) {
        case 1: return launch_T3<1>(m0, m1, a, B, qoff, resid, st);
        case 2: return launch_T3<2>(m0, m1, a, B, qoff, resid, st);
        case 3: return launch_T3<3>(m0, m1, a, B, qoff, resid, st);
        case 4: return launch_T3<4>(m0, m1, a, B, qoff, resid, st);
        case 5: return launch_T3<5>(m0, m1, a, B, qoff, resid, st);
        case 6: return launch_T3<6>(m0, m1, a, B, qoff, resid, st);
        case 7: return launch_T3<7>(m0, m1, a, B, qoff, resid, st);
        case 8: return launch_T3<8>(m0, m1, a, B, qoff, resid, st);
        default: return cudaErrorInvalidValue;
    }
}

// Force module loading of every relaxation kernel instance (CUDA lazy loading would otherwise put a
// millisecond-scale load inside the first launch of each instance).
template <int T>
static void preload_T() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_rb_tblock<T, 0, false>);
    cudaFuncGetAttributes(&a, k_rb_tblock<T, 0, true>);
    cudaFuncGetAttributes(&a, k_rb_tblock<T, 1, false>);
    cudaFuncGetAttributes(&a, k_rb_tblock<T, 1, true>);
}

void preload_relax_kernels() {
    preload_T<1>(); preload_T<2>(); preload_T<3>(); preload_T<4>();
    preload_T<5>(); preload_T<6>(); preload_T<7>(); preload_T<8>();
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_lex);
    cudaFuncGetAttributes(&a, k_jacobi);
    cudaFuncGetAttributes(&a, k_check);
    cudaFuncGetAttributes(&a, k_relax_init);
    cudaFuncGetAttributes(&a, k_fixup);
    cudaFuncGetAttributes(&a, k_res_group_max);
    cudaFuncGetAttributes(&a, k_rb_small);
    cudaGetLastError();
}

cudaError_t launch_check(int B, int* done, int* sweeps, unsigned* res_bits, float* res_final, int* where, int chunk,
                         int check_every, int max_sweeps, float tol, const int* cur, int lp, cudaStream_t st) {
    cudaError_t e = launch_pdl(k_check, dim3((B + 127) / 128), dim3(128), 0, st, B, done, sweeps, res_bits, res_final,
                               where, chunk, check_every, max_sweeps, tol, cur, lp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_fixup(float* u0, float* u1, int64_t sstride, int B, const int* where, const int* cur, int lp,
                         cudaStream_t st) {
    dim3 grid(256, B);
    k_fixup<<<grid, 256, 0, st>>>(u0, u1, sstride, where, cur, lp);
    return cudaGetLastError();
}

}  // namespace twg
