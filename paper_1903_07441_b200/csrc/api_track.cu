// api_track.cu -- row f1 entry points: the device tracker tick and its resident track table.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "api_host.cuh"

using namespace twg;
using namespace twg::host;


TWG_API twg_status twg_track_update(twg_ctx* c, int32_t b, const double* det_xy, const int32_t* n_det,
                                    const twg_warp_cfg* wc, const twg_tracker_cfg* cfg, int32_t* n_tracks) {
    TWG_NVTX("twg_track_update");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!n_det || !wc || !cfg || b < -1 || b >= c->B) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    if (!(cfg->sigma_z >= 0.0) || !(cfg->gate >= 0.0) || !(cfg->spawn_var_pos >= 0.0) || !(cfg->spawn_var_vel >= 0.0) ||
        cfg->prune_after < 0 || cfg->max_tracks < 0)
        return fail(c, TWG_E_INVALID_ARG, "tracker cfg: sigma_z, gate, variances >= 0, prune_after, max_tracks >= 0");
    const int nreq = b < 0 ? c->B : 1;
    std::vector<TrkReq> rq(nreq);
    int64_t total = 0;
    for (int k = 0; k < nreq; ++k) {
        if (n_det[k] < 0) return fail(c, TWG_E_INVALID_ARG, "negative detection count");
        rq[k].b = b < 0 ? k : b;
        rq[k].n = c->scen[rq[k].b].trk_n;
        rq[k].m = n_det[k];
        rq[k].det_off = total;
        total += n_det[k];
    }
    if (total > 0 && !det_xy) return fail(c, TWG_E_INVALID_ARG, "null detections");
    // detections -> device (double2)
    const double2* det = nullptr;
    if (total > 0) {
        if (is_device_ptr(det_xy) && (reinterpret_cast<uintptr_t>(det_xy) & 15) == 0) {
            det = reinterpret_cast<const double2*>(det_xy);
        } else {
            if (c->trk_det_cap < total) {
                if (c->d_trk_det) cudaFree(c->d_trk_det);
                c->d_trk_det = nullptr;
                TWG_CUDA(c, dev_alloc(&c->d_trk_det, (size_t)total));
                c->trk_det_cap = total;
            }
            if (is_device_ptr(det_xy)) {
                TWG_CUDA(c, cudaMemcpyAsync(c->d_trk_det, det_xy, (size_t)total * sizeof(double2),
                                            cudaMemcpyDeviceToDevice, c->stream));
            } else {
                void* hd = nullptr;
                TWG_CUDA(c, stage_alloc(c, (size_t)total * sizeof(double2), &hd));
                std::memcpy(hd, det_xy, (size_t)total * sizeof(double2));
                TWG_CUDA(c, cudaMemcpyAsync(c->d_trk_det, hd, (size_t)total * sizeof(double2), cudaMemcpyHostToDevice,
                                            c->stream));
            }
            det = c->d_trk_det;
        }
    }
    std::vector<int> nout;
    st = track_core(c, rq, det, wc, cfg, nout);
    if (st < 0) return st;
    if (n_tracks)
        for (int k = 0; k < nreq; ++k) n_tracks[k] = nout[k];
    return st;
}

TWG_API twg_status twg_get_tracks(twg_ctx* c, int32_t b, twg_track* out, int32_t* missed, int32_t cap, int32_t* n) {
    TWG_NVTX("twg_get_tracks");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (b < 0 || b >= c->B || cap < 0) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    const int nt = c->scen[b].trk_n;
    if (n) *n = nt;
    const int k = std::min(cap, nt);
    if (k > 0) {
        const int64_t o = (int64_t)b * c->track_cap;
        if (out)
            TWG_CUDA(c, cudaMemcpyAsync(out, c->d_tracks + o, k * sizeof(twg_track), cudaMemcpyDefault, c->stream));
        if (missed)
            TWG_CUDA(c, cudaMemcpyAsync(missed, c->d_missed + o, k * sizeof(int), cudaMemcpyDefault, c->stream));
    }
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

