// fgmatte::ml_foreground_background on the B200 path: a drop-in for
// proj/src/multilevel.cpp (link this TU instead of it, plus
// libfgmatte_b200.so).  The reference's Image containers and resize
// (src/image.cpp) are kept; the solve goes through the C ABI
// (include/fgmatte_b200.h).  See INTEGRATION.md.
#include <array>
#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fgmatte/multilevel.hpp"
#include "fgmatte_b200.h"

namespace fgmatte {
namespace {

fgm_params to_c(const MlParams& p) { return {p.eps_r, p.omega, p.iters_low, p.iters_high, p.low_res_threshold}; }

void raise(int rc) {
    if (rc == FGM_INVALID_ARGUMENT) throw std::invalid_argument(fgm_last_error());
    if (rc != FGM_OK) throw std::runtime_error(fgm_last_error());
}

// One pixel on the host (test helper; multilevel.cpp:48-79 contract), through
// the reference header's own PixelSystem (multilevel.hpp:45-75: init, one
// add_neighbor per neighbour, determinant, solve_raw with 1 / det), so the
// result is bitwise the reference's.  Errors as the reference:
// invalid_argument for bad parameters or neighbour lists, runtime_error for a
// singular system.
PixelSolution solve_one(double ai, const std::array<double, 3>& in, const std::vector<double>& na,
                        const std::vector<std::array<double, 3>>& nf, const std::vector<std::array<double, 3>>& nb,
                        const MlParams& params, bool clamp) {
    params.validate();
    const std::size_t n = na.size();
    if (n < 1) throw std::invalid_argument("solve_pixel: at least one neighbor required");
    if (nf.size() != n || nb.size() != n) throw std::invalid_argument("solve_pixel: neighbor lists must share length");
    PixelSystem sys;
    sys.init(ai, in.data());
    for (std::size_t j = 0; j < n; ++j)
        sys.add_neighbor(params.eps_r + params.omega * std::abs(ai - na[j]), nf[j].data(), nb[j].data());
    const double det = sys.determinant();
    if (!(det > 0.0) || !std::isfinite(1.0 / det))
        throw std::runtime_error("solve_pixel: singular 2x2 system (det = " + std::to_string(det) + ")");
    PixelSolution sol;
    sys.solve_raw(1.0 / det, sol.fg.data(), sol.bg.data());
    if (clamp)
        for (int c = 0; c < 3; ++c) {
            sol.fg[std::size_t(c)] = clamp01(sol.fg[std::size_t(c)]);
            sol.bg[std::size_t(c)] = clamp01(sol.bg[std::size_t(c)]);
        }
    return sol;
}

}  // namespace

void MlParams::validate() const {  // multilevel.cpp:10-15, same messages
    const fgm_params c = to_c(*this);
    raise(fgm_params_validate(&c));
}

LevelSchedule level_schedule(int w, int h, const MlParams& params) {  // multilevel.cpp:17-44
    const fgm_params c = to_c(params);
    int lw[64], lh[64], it[64];
    const int n = fgm_level_schedule(w, h, &c, lw, lh, it, 64);
    if (n < 0) raise(-n);
    LevelSchedule s;
    for (int l = 0; l < n; ++l) s.levels.push_back({lw[l], lh[l], it[l]});
    return s;
}

PixelSolution solve_pixel(double alpha_i, const std::array<double, 3>& intensity,
                          const std::vector<double>& neighbor_alphas,
                          const std::vector<std::array<double, 3>>& neighbor_fg,
                          const std::vector<std::array<double, 3>>& neighbor_bg, const MlParams& params) {
    return solve_one(alpha_i, intensity, neighbor_alphas, neighbor_fg, neighbor_bg, params, true);
}

PixelSolution solve_pixel_raw(double alpha_i, const std::array<double, 3>& intensity,
                              const std::vector<double>& neighbor_alphas,
                              const std::vector<std::array<double, 3>>& neighbor_fg,
                              const std::vector<std::array<double, 3>>& neighbor_bg, const MlParams& params) {
    return solve_one(alpha_i, intensity, neighbor_alphas, neighbor_fg, neighbor_bg, params, false);
}

std::pair<Image, Image> ml_foreground_background(const Image& image, const AlphaMatte& alpha,
                                                 const MlParams& params) {  // multilevel.cpp:141-166
    params.validate();
    if (image.channels() != 3)
        throw std::invalid_argument("ml_foreground_background: image must have 3 channels, got " +
                                    std::to_string(image.channels()));
    if (image.width() != alpha.width() || image.height() != alpha.height())
        throw std::invalid_argument("ml_foreground_background: alpha size " + std::to_string(alpha.width()) + "x" +
                                    std::to_string(alpha.height()) + " does not match image size " +
                                    std::to_string(image.width()) + "x" + std::to_string(image.height()));
    Image fg(image.width(), image.height(), 3), bg(image.width(), image.height(), 3);
    const fgm_params c = to_c(params);
    raise(fgm_ml_solve_host_f64(image.data().data(), alpha.data().data(), image.width(), image.height(), &c,
                                fg.data().data(), bg.data().data()));
    return {std::move(fg), std::move(bg)};
}

}  // namespace fgmatte
