// TEST INFRASTRUCTURE ONLY: an extern "C" shim over the UNMODIFIED reference
// library (fgmatte, /root/reference/proj/src/{image,multilevel}.cpp), compiled
// from the reference sources where they lie by oracle/Makefile into
// oracle/_ref/libfgmatte_ref.so.  Nothing here restates the algorithm: every
// entry point converts planar arrays into the reference's own containers and
// calls the reference function named in its comment.  Used to pin the C
// restatement (fgm_oracle.c) and as the timed CPU baseline in bench.py.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fgmatte/image.hpp"
#include "fgmatte/metrics.hpp"
#include "fgmatte/multilevel.hpp"

using namespace fgmatte;

namespace {
thread_local std::string g_err;

MlParams make_params(double omega, double eps_r, int thr, int il, int ih) {
    MlParams p;  // multilevel.hpp:12-20
    p.omega = omega;
    p.eps_r = eps_r;
    p.low_res_threshold = thr;
    p.iters_low = il;
    p.iters_high = ih;
    return p;
}

int run_guarded(const std::function<void()>& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
}  // namespace

extern "C" {

const char* fgmr_last_error() { return g_err.c_str(); }

// fgmatte::level_schedule, multilevel.cpp:17-44
int fgmr_level_schedule(int w, int h, double omega, double eps_r, int thr, int il, int ih, int* ow, int* oh,
                        int* oit, int cap) {
    int n = -1;
    int rc = run_guarded([&] {
        const LevelSchedule s = level_schedule(w, h, make_params(omega, eps_r, thr, il, ih));
        n = int(s.levels.size());
        for (int l = 0; l < n && l < cap; ++l) {
            ow[l] = s.levels[size_t(l)].width;
            oh[l] = s.levels[size_t(l)].height;
            oit[l] = s.levels[size_t(l)].iterations;
        }
    });
    return rc ? -rc : n;
}

// fgmatte::resize(Image / AlphaMatte), image.cpp:114-133
int fgmr_resize(const double* src, int sw, int sh, int nch, double* dst, int dw, int dh) {
    return run_guarded([&] {
        const size_t sn = size_t(sw) * sh, dn = size_t(dw) * dh;
        if (nch == 1) {
            AlphaMatte a(sw, sh);
            std::memcpy(a.data().data(), src, sizeof(double) * sn);
            const AlphaMatte r = resize(a, dw, dh);
            std::memcpy(dst, r.data().data(), sizeof(double) * dn);
        } else {
            Image img(sw, sh, nch);
            std::memcpy(img.data().data(), src, sizeof(double) * sn * size_t(nch));
            const Image r = resize(img, dw, dh);
            std::memcpy(dst, r.data().data(), sizeof(double) * dn * size_t(nch));
        }
    });
}

// fgmatte::compose, image.cpp:39-57 (planar fg/bg with nch channels, alpha w*h)
int fgmr_compose(const double* fg, const double* bg, const double* alpha, int w, int h, int nch, double* out) {
    return run_guarded([&] {
        const size_t n = size_t(w) * h;
        Image f(w, h, nch), b(w, h, nch);
        AlphaMatte a(w, h);
        std::memcpy(f.data().data(), fg, sizeof(double) * n * size_t(nch));
        std::memcpy(b.data().data(), bg, sizeof(double) * n * size_t(nch));
        std::memcpy(a.data().data(), alpha, sizeof(double) * n);
        const Image o = compose(f, b, a);
        std::memcpy(out, o.data().data(), sizeof(double) * n * size_t(nch));
    });
}

// fgmatte::evaluate_metrics, metrics.cpp:75-145 (SAD, MSE, GRAD, translucent count)
int fgmr_metrics(const double* est, const double* gt, const double* alpha, int w, int h, int nch, double sigma,
                 int kernel_radius, double* out4) {
    return run_guarded([&] {
        const size_t n = size_t(w) * h;
        Image e(w, h, nch), g(w, h, nch);
        AlphaMatte a(w, h);
        std::memcpy(e.data().data(), est, sizeof(double) * n * size_t(nch));
        std::memcpy(g.data().data(), gt, sizeof(double) * n * size_t(nch));
        std::memcpy(a.data().data(), alpha, sizeof(double) * n);
        GradParams gp;
        gp.sigma = sigma;
        gp.kernel_radius = kernel_radius;
        const MetricReport r = evaluate_metrics(e, g, a, gp);
        out4[0] = r.sad;
        out4[1] = r.mse;
        out4[2] = r.grad;
        out4[3] = double(r.translucent_pixel_count);
    });
}

// fgmatte::solve_pixel / solve_pixel_raw, multilevel.cpp:125-139
int fgmr_solve_pixel(double alpha_i, const double* intensity, int n, const double* nalpha, const double* nfg,
                     const double* nbg, double omega, double eps_r, int clamp, double* fg_out, double* bg_out) {
    return run_guarded([&] {
        std::vector<double> na(nalpha, nalpha + n);
        std::vector<std::array<double, 3>> f(static_cast<size_t>(n)), b(static_cast<size_t>(n));
        for (int j = 0; j < n; ++j)
            for (int c = 0; c < 3; ++c) {
                f[size_t(j)][size_t(c)] = nfg[3 * j + c];
                b[size_t(j)][size_t(c)] = nbg[3 * j + c];
            }
        MlParams p;
        p.omega = omega;
        p.eps_r = eps_r;
        const std::array<double, 3> in = {intensity[0], intensity[1], intensity[2]};
        const PixelSolution s = clamp ? solve_pixel(alpha_i, in, na, f, b, p) : solve_pixel_raw(alpha_i, in, na, f, b, p);
        for (int c = 0; c < 3; ++c) {
            fg_out[c] = s.fg[size_t(c)];
            bg_out[c] = s.bg[size_t(c)];
        }
    });
}

// fgmatte::ml_foreground_background, multilevel.cpp:141-166.  *seconds gets the
// steady_clock time of the reference call only (as tools/main.cpp:233-249).
int fgmr_ml_solve(const double* image, const double* alpha, int w, int h, double omega, double eps_r, int thr,
                  int il, int ih, double* fg, double* bg, double* seconds) {
    return run_guarded([&] {
        Image img(w, h, 3);
        AlphaMatte a(w, h);
        const size_t n = size_t(w) * h;
        std::memcpy(img.data().data(), image, sizeof(double) * 3 * n);
        std::memcpy(a.data().data(), alpha, sizeof(double) * n);
        const MlParams p = make_params(omega, eps_r, thr, il, ih);
        const auto t0 = std::chrono::steady_clock::now();
        auto [f, b] = ml_foreground_background(img, a, p);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(fg, f.data().data(), sizeof(double) * 3 * n);
        std::memcpy(bg, b.data().data(), sizeof(double) * 3 * n);
    });
}

// The same reference call over a batch of independent images on `nthreads`
// host threads (the function is reentrant).  Images are taken
// largest-first.  Inputs are fp32 planar (as the GPU path sees them) and are
// upcast exactly to the reference's fp64 containers before the clock starts;
// outputs (optional, may be NULL) are written back as fp32.  Returns 0 and the
// wall time of the solves in *seconds.
int fgmr_ml_solve_batch_f32(int n_images, const float* const* images, const float* const* alphas, const int* ws,
                            const int* hs, double omega, double eps_r, int thr, int il, int ih, float* const* fgs,
                            float* const* bgs, int nthreads, double* seconds) {
    return run_guarded([&] {
        const MlParams p = make_params(omega, eps_r, thr, il, ih);
        std::vector<Image> imgs;
        std::vector<AlphaMatte> alps;
        imgs.reserve(size_t(n_images));
        alps.reserve(size_t(n_images));
        for (int i = 0; i < n_images; ++i) {
            const size_t n = size_t(ws[i]) * hs[i];
            imgs.emplace_back(ws[i], hs[i], 3);
            alps.emplace_back(ws[i], hs[i]);
            for (size_t k = 0; k < 3 * n; ++k) imgs.back().data()[k] = double(images[i][k]);
            for (size_t k = 0; k < n; ++k) alps.back().data()[k] = double(alphas[i][k]);
        }
        std::vector<int> order(static_cast<size_t>(n_images));
        for (int i = 0; i < n_images; ++i) order[size_t(i)] = i;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
            return size_t(ws[a]) * hs[a] > size_t(ws[b]) * hs[b];
        });
        std::atomic<int> next{0};
        std::vector<std::string> errs(size_t(std::max(1, nthreads)));
        auto worker = [&](int tid) {
            try {
                for (;;) {
                    const int k = next.fetch_add(1);
                    if (k >= n_images) break;
                    const int i = order[size_t(k)];
                    auto [f, b] = ml_foreground_background(imgs[size_t(i)], alps[size_t(i)], p);
                    if (fgs && fgs[i]) {
                        const size_t n = size_t(ws[i]) * hs[i];
                        for (size_t q = 0; q < 3 * n; ++q) {
                            fgs[i][q] = float(f.data()[q]);
                            bgs[i][q] = float(b.data()[q]);
                        }
                    }
                }
            } catch (const std::exception& e) {
                errs[size_t(tid)] = e.what();
            }
        };
        const int nt = std::max(1, nthreads);
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(worker, t);
        worker(0);
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (const auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

}  // extern "C"
