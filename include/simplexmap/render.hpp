// Drop-in forwarding header: `#include <simplexmap/render.hpp>` with -I<repo>/include
// resolves to the B200 implementation (include/simplexmap_b200.hpp, exposed as
// namespace simplexmap) instead of the reference's
// /root/reference/proj/include/simplexmap/render.hpp.
#pragma once
#ifndef SMX_B200_AS_SIMPLEXMAP
#define SMX_B200_AS_SIMPLEXMAP 1
#endif
#include "../simplexmap_b200.hpp"
