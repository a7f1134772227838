// api_sim.cu -- row f2 entry points: the batched closed-loop simulator around Algorithm 1.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "api_host.cuh"

using namespace twg;
using namespace twg::host;

namespace {
// Simulator buffers with room for `ocap` obstacles per trial (contents kept when growing).
twg_status ensure_sim(twg_ctx* c, int ocap) {
    const size_t B = c->B;
    if (!c->d_sim_rob) {
        TWG_CUDA(c, dev_alloc(&c->d_sim_rob, B * 6));
        TWG_CUDA(c, dev_alloc(&c->d_sim_int, B * 2));
        TWG_CUDA(c, dev_alloc(&c->d_sim_goal, B * 2));
        TWG_CUDA(c, dev_alloc(&c->d_sim_nobs, B));
        TWG_CUDA(c, dev_alloc(&c->d_sim_hist, B * 36));
        c->sim_rob.assign(B * 6, 0.0);
        c->sim_ticks.assign(B, 0);
        c->sim_status.assign(B, 4);
        c->sim_nobs.assign(B, 0);
        std::vector<int> init(2 * B, 0);
        for (size_t b = 0; b < B; ++b) init[B + b] = 4;  // idle
        TWG_CUDA(c, cudaMemcpy(c->d_sim_int, init.data(), 2 * B * sizeof(int), cudaMemcpyHostToDevice));
        TWG_CUDA(c, cudaMemset(c->d_sim_nobs, 0, B * sizeof(int)));
    }
    if (ocap <= c->sim_ocap) return TWG_OK;
    const int nc = std::max(ocap, std::max(2 * c->sim_ocap, 16));
    double *o, *oo, *sp;
    double2* dt;
    TWG_CUDA(c, dev_alloc(&o, B * nc * 4));
    TWG_CUDA(c, dev_alloc(&oo, B * nc * 4));
    TWG_CUDA(c, dev_alloc(&sp, B * nc));
    TWG_CUDA(c, dev_alloc(&dt, B * nc));
    if (c->sim_ocap > 0) {
        const int oc = c->sim_ocap;
        TWG_CUDA(c, cudaMemcpy2DAsync(o, nc * 4 * sizeof(double), c->d_sim_obs, oc * 4 * sizeof(double),
                                      oc * 4 * sizeof(double), B, cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaMemcpy2DAsync(sp, nc * sizeof(double), c->d_sim_speed, oc * sizeof(double), oc * sizeof(double),
                                      B, cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaMemcpy2DAsync(dt, nc * sizeof(double2), c->d_sim_det, oc * sizeof(double2),
                                      oc * sizeof(double2), B, cudaMemcpyDeviceToDevice, c->stream));
        TWG_CUDA(c, cudaStreamSynchronize(c->stream));
        cudaFree(c->d_sim_obs);
        cudaFree(c->d_sim_obs_old);
        cudaFree(c->d_sim_speed);
        cudaFree(c->d_sim_det);
    }
    c->d_sim_obs = o;
    c->d_sim_obs_old = oo;
    c->d_sim_speed = sp;
    c->d_sim_det = dt;
    c->sim_ocap = nc;
    return TWG_OK;
}

bool sim_cfg_ok(const twg_sim_cfg* f) {
    return f && f->dt > 0.0 && f->robot_radius >= 0.0 && f->obstacle_radius >= 0.0 && f->goal_radius >= 0.0 &&
           f->turn_distance >= 0.0 && f->heading_sigma >= 0.0 && f->det_sigma >= 0.0 && f->turn_max >= 0.0 &&
           f->max_ticks > 0 && f->init_max_sweeps >= 0;
}

SimArgs sim_args(twg_ctx* c, const twg_sim_cfg* f) {
    SimArgs a;
    a.B = c->B;
    a.W = c->W;
    a.H = c->H;
    a.ocap = c->sim_ocap;
    a.cs = c->cs;
    a.ox = c->ox;
    a.oy = c->oy;
    a.mask = c->mask;
    a.rob = c->d_sim_rob;
    a.ticks = c->d_sim_int;
    a.status = c->d_sim_int + c->B;
    a.goal = c->d_sim_goal;
    a.n_obs = c->d_sim_nobs;
    a.obs = c->d_sim_obs;
    a.obs_old = c->d_sim_obs_old;
    a.obs_speed = c->d_sim_speed;
    a.det = c->d_sim_det;
    a.hist = c->d_sim_hist;
    a.meta = c->d_meta;
    a.dt = f->dt;
    a.r_robot = f->robot_radius;
    a.r_obs = f->obstacle_radius;
    a.goal_r = f->goal_radius;
    a.turn_dist = f->turn_distance;
    a.sigma_h = f->heading_sigma;
    a.sigma_z = f->det_sigma;
    a.cos_d = std::cos(f->turn_max);  // host libm (C25)
    a.sin_d = std::sin(f->turn_max);
    for (int k = 0; k < 37; ++k) a.cos_bins[k] = std::cos(k * 5.0 * M_PI / 180.0);
    a.seed = f->seed;
    a.max_ticks = f->max_ticks;
    return a;
}
}  // namespace

TWG_API twg_status twg_sim_reset(twg_ctx* c, int32_t b, const twg_robot* robot, int32_t goal_x, int32_t goal_y,
                                 const double* obstacles, int32_t n, const twg_sim_cfg* cfg) {
    TWG_NVTX("twg_sim_reset");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!robot || b < 0 || b >= c->B || n < 0 || (n > 0 && !obstacles) || !sim_cfg_ok(cfg))
        return fail(c, TWG_E_INVALID_ARG, "bad argument");
    if (c->ghost > 0) return fail(c, TWG_E_INVALID_ARG, "the simulator is not available on a row slab");
    st = ensure_sim(c, std::max(n, 1));
    if (st != TWG_OK) return st;
    // Alg. 1 "Initialize the 2D map and harmonic potential values" (C36): static map + goal,
    // no tracks, cold, relaxed to init_tol (checked every 100 sweeps)
    EncodeReq r{b, *robot, goal_x, goal_y, 0, 0};
    c->scen[b].encoded = false;
    twg_warp_cfg wz;  // no tracks: the warp configuration is not used
    std::memset(&wz, 0, sizeof(wz));
    st = encode(c, {r}, nullptr, &wz, 0);
    if (st < 0) return st;
    std::vector<int> part(c->B, 0);
    part[b] = 1;
    twg_relax_cfg rc;
    std::memset(&rc, 0, sizeof(rc));
    rc.max_sweeps = cfg->init_max_sweeps;
    rc.check_every = 100;
    rc.tol = cfg->init_tol;
    st = relax(c, &rc, part, nullptr, nullptr);
    if (st != TWG_OK) return st;
    // trial state
    const int oc = c->sim_ocap;
    char* h = nullptr;
    const size_t bytes = 6 * sizeof(double) + 2 * sizeof(double) + (size_t)oc * 5 * sizeof(double);
    TWG_CUDA(c, stage_alloc(c, bytes, reinterpret_cast<void**>(&h)));
    double* hr = reinterpret_cast<double*>(h);
    hr[0] = robot->x;
    hr[1] = robot->y;
    hr[2] = std::cos(robot->theta);  // host libm (C25)
    hr[3] = std::sin(robot->theta);
    hr[4] = robot->speed;
    hr[5] = 0.0;
    double* hg = hr + 6;
    hg[0] = c->ox + ((double)goal_x + 0.5) * c->cs;
    hg[1] = c->oy + ((double)goal_y + 0.5) * c->cs;
    double* ho = hg + 2;
    double* hs = ho + (size_t)oc * 4;
    std::memset(ho, 0, (size_t)oc * 5 * sizeof(double));
    for (int i = 0; i < n; ++i) {
        for (int q = 0; q < 4; ++q) ho[4 * i + q] = obstacles[4 * i + q];
        hs[i] = std::sqrt(obstacles[4 * i + 2] * obstacles[4 * i + 2] + obstacles[4 * i + 3] * obstacles[4 * i + 3]);
    }
    TWG_CUDA(c, cudaMemcpyAsync(c->d_sim_rob + 6 * b, hr, 6 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    TWG_CUDA(c, cudaMemcpyAsync(c->d_sim_goal + 2 * b, hg, 2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    TWG_CUDA(c, cudaMemcpyAsync(c->d_sim_obs + (size_t)b * oc * 4, ho, (size_t)oc * 4 * sizeof(double),
                                cudaMemcpyHostToDevice, c->stream));
    TWG_CUDA(c, cudaMemcpyAsync(c->d_sim_speed + (size_t)b * oc, hs, (size_t)oc * sizeof(double),
                                cudaMemcpyHostToDevice, c->stream));
    TWG_CUDA(c, cudaMemsetAsync(c->d_sim_int + b, 0, sizeof(int), c->stream));          // ticks
    TWG_CUDA(c, cudaMemsetAsync(c->d_sim_int + c->B + b, 0, sizeof(int), c->stream));   // running
    TWG_CUDA(c, cudaMemsetAsync(c->d_sim_hist + 36 * b, 0, 36 * sizeof(int), c->stream));
    int* hn = nullptr;
    TWG_CUDA(c, stage_alloc(c, sizeof(int), reinterpret_cast<void**>(&hn)));
    *hn = n;
    TWG_CUDA(c, cudaMemcpyAsync(c->d_sim_nobs + b, hn, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    SimArgs a = sim_args(c, cfg);
    TWG_CUDA(c, launch_sim_sense(a, b, c->stream));
    c->launches += 1;
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int q = 0; q < 6; ++q) c->sim_rob[6 * b + q] = hr[q];
    c->sim_ticks[b] = 0;
    c->sim_status[b] = 0;
    c->sim_nobs[b] = n;
    c->scen[b].trk_n = 0;
    return TWG_OK;
}

TWG_API twg_status twg_sim_tick(twg_ctx* c, const twg_sim_cfg* cfg, const twg_warp_cfg* warp,
                                const twg_relax_cfg* rcfg, const twg_band_cfg* bcfg, const twg_tracker_cfg* tcfg,
                                twg_sim_trial* out, int32_t* running) {
    TWG_NVTX("twg_sim_tick");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!sim_cfg_ok(cfg) || !warp || !rcfg || !bcfg || !tcfg) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    if (!c->d_sim_rob) return fail(c, TWG_E_INVALID_ARG, "twg_sim_tick before twg_sim_reset");
    std::vector<int> act;
    for (int b = 0; b < c->B; ++b)
        if (c->sim_status[b] == 0) act.push_back(b);
    int worst = 0;
    if (!act.empty()) {
        // f1: tracker tick on this tick's detections
        std::vector<TrkReq> rq(act.size());
        for (size_t k = 0; k < act.size(); ++k) {
            const int b = act[k];
            rq[k].b = b;
            rq[k].n = c->scen[b].trk_n;
            rq[k].m = c->sim_nobs[b];
            rq[k].det_off = (int64_t)b * c->sim_ocap;
        }
        std::vector<int> nout;
        st = track_core(c, rq, c->d_sim_det, warp, tcfg, nout);
        if (st < 0) return st;
        worst = std::max(worst, (int)st);
        // a1-a9 from the resident tracks
        std::vector<EncodeReq> reqs;
        for (int b : act) {
            twg_robot rb;
            rb.x = c->sim_rob[6 * b];
            rb.y = c->sim_rob[6 * b + 1];
            rb.theta = std::atan2(c->sim_rob[6 * b + 3], c->sim_rob[6 * b + 2]);  // host libm (C25)
            rb.speed = c->sim_rob[6 * b + 4];
            reqs.push_back(EncodeReq{b, rb, c->scen[b].gx, c->scen[b].gy, c->scen[b].trk_n, 0});
        }
        st = encode(c, reqs, nullptr, warp, rcfg->warm_start, true);
        if (st < 0) return st;
        std::vector<int> part(c->B, 0);
        for (int b : act) part[b] = 1;
        st = relax(c, rcfg, part, nullptr, nullptr);
        if (st != TWG_OK) return st;
        st = path(c, act, bcfg);
        if (st != TWG_OK) return st;
        // simulator step + next detections
        SimArgs a = sim_args(c, cfg);
        TWG_CUDA(c, launch_sim_move(a, c->stream));
        TWG_CUDA(c, launch_sim_sense(a, -1, c->stream));
        c->launches += 2;
    }
    // read back the trial states
    const size_t B = c->B;
    char* h = nullptr;
    TWG_CUDA(c, stage_alloc(c, B * 6 * sizeof(double) + 2 * B * sizeof(int), reinterpret_cast<void**>(&h)));
    double* hr = reinterpret_cast<double*>(h);
    int* hi = reinterpret_cast<int*>(hr + 6 * B);
    TWG_CUDA(c, cudaMemcpyAsync(hr, c->d_sim_rob, B * 6 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaMemcpyAsync(hi, c->d_sim_int, 2 * B * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    int nrun = 0;
    for (size_t b = 0; b < B; ++b) {
        for (int q = 0; q < 6; ++q) c->sim_rob[6 * b + q] = hr[6 * b + q];
        c->sim_ticks[b] = hi[b];
        c->sim_status[b] = hi[B + b];
        nrun += c->sim_status[b] == 0;
        if (out) {
            out[b].x = hr[6 * b];
            out[b].y = hr[6 * b + 1];
            out[b].hx = hr[6 * b + 2];
            out[b].hy = hr[6 * b + 3];
            out[b].speed = hr[6 * b + 4];
            out[b].length = hr[6 * b + 5];
            out[b].ticks = hi[b];
            out[b].status = hi[B + b];
        }
    }
    if (running) *running = nrun;
    return (twg_status)worst;
}

TWG_API twg_status twg_sim_histogram(twg_ctx* c, int32_t b, int32_t* hist) {
    TWG_NVTX("twg_sim_histogram");
    twg_status st = check_ctx(c);
    if (st != TWG_OK) return st;
    if (!hist || b < 0 || b >= c->B || !c->d_sim_hist) return fail(c, TWG_E_INVALID_ARG, "bad argument");
    TWG_CUDA(c, cudaMemcpyAsync(hist, c->d_sim_hist + 36 * b, 36 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    TWG_CUDA(c, cudaStreamSynchronize(c->stream));
    return TWG_OK;
}

