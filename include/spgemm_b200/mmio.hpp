// spgemm_b200/mmio.hpp — Matrix Market I/O with the reference's semantics
// (proj/include/spgemm/mmio.hpp:15-21, mmio.cpp:33-117), backed by the host
// library (include/pbg_host.h pbgh_mm_*): coordinate real/integer/pattern,
// general/symmetric (expanded), 1-based in, 0-based out; malformed input
// throws parse_error with the reference's "name:line: what" message.
#pragma once

#include <string>

#include "spgemm_b200/types.hpp"

namespace spgemm {

CooMatrix mm_read(const std::string& path);
void mm_write(const CooMatrix& m, const std::string& path);

}  // namespace spgemm
