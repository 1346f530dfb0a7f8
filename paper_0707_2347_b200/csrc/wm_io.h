// Matrix file formats (ring.hpp:386-449), host side (wm_io.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "wm_types.h"

namespace wm {

struct MatrixFile {
    std::uint64_t rows = 0, cols = 0;
    std::uint32_t p = 0;
    std::vector<std::uint32_t> data;  // row-major residues (empty when header_only)
    std::size_t body = 0;
};

// read_text / read_binary (ring.hpp:401-446); E_IO on a bad header, a truncated
// body or a non-canonical entry
MatrixFile read_matrix_file(const char* path, bool binary, bool header_only = false);
// write_text / write_binary (ring.hpp:390-434)
void write_matrix_file(const char* path, bool binary, std::uint64_t rows, std::uint64_t cols,
                       std::uint32_t p, const std::uint32_t* data);

}  // namespace wm
