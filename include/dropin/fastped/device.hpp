// Device plumbing shared by the drop-in overlay headers (include/dropin/fastped/*.hpp): error
// mapping from the C ABI status codes to the reference's exception types, the device ordinal,
// and Grid -> fp_grid_desc conversion.  Not a reference header; included only by the overlay.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../fastped_b200.h"

namespace fastped {
class Grid;
namespace b200 {

/// CUDA ordinal every drop-in SimState uses (env FASTPED_B200_DEVICE, default 0).
inline int& device() {
    static int d = [] {
        const char* e = std::getenv("FASTPED_B200_DEVICE");
        return e ? std::atoi(e) : 0;
    }();
    return d;
}

/// FP_EINVAL -> std::invalid_argument (the reference's validation errors, same wording);
/// everything else (runtime, CUDA, NCCL) -> std::runtime_error.  No CPU fallback.
[[noreturn]] inline void raise(int code, const fp_ctx* ctx) {
    const std::string msg = fp_last_error(ctx);
    if (code == FP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
inline void check(int code, const fp_ctx* ctx = nullptr) {
    if (code != FP_OK) raise(code, ctx);
}

template <class G>
inline fp_grid_desc desc_of(const G& g) {
    return fp_grid_desc{g.width(), g.height(), g.cell_size(), static_cast<std::int32_t>(g.boundary())};
}

template <class G>
inline std::vector<std::uint8_t> cells_of(const G& g) {
    std::vector<std::uint8_t> c(static_cast<std::size_t>(g.width()) * static_cast<std::size_t>(g.height()));
    std::size_t i = 0;
    for (int y = 0; y < g.height(); ++y)
        for (int x = 0; x < g.width(); ++x) c[i++] = static_cast<std::uint8_t>(g.at(x, y));
    return c;
}

}  // namespace b200
}  // namespace fastped
