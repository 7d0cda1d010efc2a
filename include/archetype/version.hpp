// Library version string (drop-in for
// /root/reference/proj/include/archetype/version.hpp:5). report.json carries it.
#pragma once

namespace archetype {

inline constexpr const char* kVersion = "0.1.0";

}  // namespace archetype
