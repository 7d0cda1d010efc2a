// ENVI BSQ cube reader (drop-in for /root/reference/proj/include/archetype/envi.hpp:9-17;
// behaviour of src/envi.cpp:101-179). Supported subset: interleave bsq, data
// type 4 (f32) or 5 (f64), byte order 0; anything else names the field.
#pragma once

#include <string>

#include "archetype/image.hpp"

namespace archetype {

/// Header + raw band-sequential payload → L×(lines·samples) image with the
/// spatial grid and, when listed, the wavelengths.
HsiImage read_envi(const std::string& header_path, const std::string& data_path);

/// The data file next to a header: the path without ".hdr", or that base
/// plus ".img" / ".dat" / ".raw", first that exists.
std::string envi_data_path(const std::string& header_path);

}  // namespace archetype
