// Drop-in overlay of fastped/world.hpp (/root/reference/proj/include/fastped/world.hpp).
//
// Put include/dropin BEFORE the reference's include directory:
//     g++ -std=c++20 -I<repo>/include/dropin -I<reference>/proj/include ...
// Every `#include "fastped/X.hpp"` then resolves here first.  This file keeps the reference's
// geometry types unchanged (Grid, Cell, StaticField, segment_dx, walk_segment, line_of_sight,
// the scenario text grammar -- world.hpp:18-406, via #include_next) and serves exactly one
// function from the device: compute_static_field (world.hpp:220-266) becomes the bit-identical
// Dial-bucketed relaxation of libfastped_b200 (fp_static_field).  The reference's CPU version
// stays reachable as compute_static_field_host.
#pragma once

#define compute_static_field compute_static_field_host
#include_next <fastped/world.hpp>
#undef compute_static_field

#include "../../fastped_b200.h"
#include "device.hpp"

namespace fastped {

/// compute_static_field(g) -- world.hpp:220-266, on the device (bitwise the reference's field).
inline StaticField compute_static_field(const Grid& g) {
    StaticField f{g.width(), g.height(),
                  std::vector<double>(static_cast<std::size_t>(g.width()) * static_cast<std::size_t>(g.height()))};
    const fp_grid_desc d = b200::desc_of(g);
    const std::vector<std::uint8_t> cells = b200::cells_of(g);
    b200::check(fp_static_field(&d, cells.data(), b200::device(), f.s.data()));
    return f;
}

}  // namespace fastped
