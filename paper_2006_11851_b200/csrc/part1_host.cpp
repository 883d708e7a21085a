// Part 1 of the pipeline: scale-matched initialisation of the coarsest output
// level, initialize_output (pipeline.cpp:96-175).
//
// Each output pixel copies the RGB of an exemplar pixel whose unnormalised
// scale lies within 1e-3 of the pixel's target scale, chosen uniformly with
// ONE std::mt19937_64 consumed in row-major pixel order; with no such pixel,
// the nearest scale (an exact distance tie takes the run holding the lowest
// row-major index).  The draws are sequential by definition (each pixel's
// draw depends on how many pixels before it drew), so this runs once per
// synthesis on the host, with the same engine / distribution types from the
// same C++ library as the reference -- identical picks by construction.  It
// is O(P log N) host work done once, ahead of the device-resident EM stages.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <utility>
#include <vector>

#include "psg_internal.h"

namespace psg {

void initialize_output_host(const double* ex_planes, int C, int ew, int eh,
                            const float* out_scale, int ow, int oh, double s_min, double s_max,
                            uint64_t seed, double* out4) {
  if (C < 4) fail(PSG_E_SHAPE, "exemplar needs an S plane (C >= 4)");
  if (ew < 1 || eh < 1 || ow < 1 || oh < 1) fail(PSG_E_DOMAIN, "empty image");
  const size_t en = (size_t)ew * eh, on = (size_t)ow * oh;
  const double* S = ex_planes + 3 * en;
  const bool spread = s_max > s_min;
  // exemplar pixels sorted by (raw scale, row-major index)
  std::vector<std::pair<double, int32_t>> key(en);
  for (size_t i = 0; i < en; ++i)
    key[i] = {spread ? s_min + S[i] * (s_max - s_min) : s_min, (int32_t)i};
  std::sort(key.begin(), key.end());
  // first entry of the run of equal scales containing position pos
  auto run_head = [&](size_t pos) {
    return std::lower_bound(key.begin(), key.end(), std::pair<double, int32_t>{key[pos].first, -1})
        ->second;
  };
  constexpr double kTol = 1e-3;
  std::mt19937_64 rng(seed);
  const double inv = spread ? 1.0 / (s_max - s_min) : 0.0;
  for (int y = 0; y < oh; ++y) {
    for (int x = 0; x < ow; ++x) {
      const size_t o = (size_t)y * ow + x;
      const double t = out_scale[o];
      const auto lo = std::lower_bound(key.begin(), key.end(),
                                       std::pair<double, int32_t>{t - kTol, -1});
      const auto hi = std::upper_bound(
          lo, key.end(), std::pair<double, int32_t>{t + kTol, std::numeric_limits<int32_t>::max()});
      int32_t src;
      if (lo != hi) {
        std::uniform_int_distribution<std::size_t> pick(0, (size_t)(hi - lo) - 1);
        src = (lo + (std::ptrdiff_t)pick(rng))->second;
      } else {
        const size_t r = (size_t)(lo - key.begin());
        if (r == 0) {
          src = run_head(0);
        } else if (r == en) {
          src = run_head(en - 1);
        } else {
          const double dl = std::abs(key[r - 1].first - t), dr = std::abs(key[r].first - t);
          src = dl < dr ? run_head(r - 1)
                        : dr < dl ? run_head(r) : std::min(run_head(r - 1), run_head(r));
        }
      }
      for (int c = 0; c < 3; ++c) out4[c * on + o] = ex_planes[c * en + (size_t)src];
      // S = the target map normalised against its bounds (normalized_plane,
      // pipeline.cpp:23-35)
      out4[3 * on + o] = spread ? std::clamp((t - s_min) * inv, 0.0, 1.0) : 0.5;
    }
  }
}

}  // namespace psg
