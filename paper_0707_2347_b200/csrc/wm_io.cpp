// Matrix file formats of the reference (ring.hpp:386-449), read straight into
// device memory and written from it:
//   text:   "rows cols p\n", then rows*cols canonical residues, row-major,
//           whitespace separated (one row per line when written);
//   binary: three little-endian u64 (rows, cols, p), then u64 residues.
// A bad header, a truncated body or a non-canonical entry is io_error (E_IO),
// as in the reference readers.  Parsing and formatting are host work over one
// buffered pass; the device side is one u32 upload / download (wm_runtime.cu).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "wm_io.h"

namespace wm {
namespace {

struct File {
    std::FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

std::vector<char> slurp(const char* path) {
    File in(path, "rb");
    if (!in.f) fail(E_IO, std::string("cannot open ") + path);
    std::vector<char> buf;
    char chunk[1 << 16];
    std::size_t n;
    while ((n = std::fread(chunk, 1, sizeof(chunk), in.f)) > 0) buf.insert(buf.end(), chunk, chunk + n);
    return buf;
}

// unsigned decimal token at *pos (leading whitespace skipped); false at end of
// data or on a non-digit (the reference's `is >> uint64` failing)
bool next_u64(const std::vector<char>& b, std::size_t* pos, std::uint64_t* v) {
    std::size_t i = *pos;
    while (i < b.size() && (b[i] == ' ' || b[i] == '\n' || b[i] == '\t' || b[i] == '\r' ||
                            b[i] == '\v' || b[i] == '\f'))
        ++i;
    if (i < b.size() && b[i] == '+') ++i;
    if (i >= b.size() || b[i] < '0' || b[i] > '9') return false;
    std::uint64_t x = 0;
    while (i < b.size() && b[i] >= '0' && b[i] <= '9') {
        const std::uint64_t d = static_cast<std::uint64_t>(b[i] - '0');
        if (x > (~0ull - d) / 10) return false;  // out of range: the stream fails
        x = x * 10 + d;
        ++i;
    }
    *pos = i;
    *v = x;
    return true;
}

std::uint64_t get_le(const std::vector<char>& b, std::size_t off) {
    std::uint64_t v = 0;
    for (int i = 0; i < 8; ++i)
        v |= static_cast<std::uint64_t>(static_cast<unsigned char>(b[off + i])) << (8 * i);
    return v;
}

}  // namespace

MatrixFile read_matrix_file(const char* path, bool binary, bool header_only) {
    const std::vector<char> b = slurp(path);
    MatrixFile m;
    std::uint64_t p = 0;
    if (binary) {
        if (b.size() < 24) fail(E_IO, "matrix binary truncated");
        m.rows = get_le(b, 0);
        m.cols = get_le(b, 8);
        p = get_le(b, 16);
    } else {
        std::size_t pos = 0;
        if (!next_u64(b, &pos, &m.rows) || !next_u64(b, &pos, &m.cols) || !next_u64(b, &pos, &p))
            fail(E_IO, "bad matrix text header");
        m.body = pos;
    }
    m.p = static_cast<std::uint32_t>(p);
    if (header_only) return m;
    const std::uint64_t count = m.rows * m.cols;
    m.data.resize(count);
    if (binary) {
        if (b.size() < 24 + 8 * count) fail(E_IO, "matrix binary truncated");
        for (std::uint64_t i = 0; i < count; ++i) {
            const std::uint64_t v = get_le(b, 24 + 8 * i);
            if (v >= p) fail(E_IO, "matrix entry not a canonical residue");
            m.data[i] = static_cast<std::uint32_t>(v);
        }
    } else {
        std::size_t pos = m.body;
        for (std::uint64_t i = 0; i < count; ++i) {
            std::uint64_t v;
            if (!next_u64(b, &pos, &v)) fail(E_IO, "matrix text truncated");
            if (v >= p) fail(E_IO, "matrix entry not a canonical residue");
            m.data[i] = static_cast<std::uint32_t>(v);
        }
    }
    return m;
}

void write_matrix_file(const char* path, bool binary, std::uint64_t rows, std::uint64_t cols,
                       std::uint32_t p, const std::uint32_t* data) {
    File out(path, binary ? "wb" : "w");
    if (!out.f) fail(E_IO, std::string("cannot open ") + path);
    std::vector<char> buf;
    buf.reserve(1 << 20);
    auto flush = [&]() {
        if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), out.f) != buf.size())
            fail(E_IO, std::string("write failed: ") + path);
        buf.clear();
    };
    auto put_le = [&](std::uint64_t v) {
        for (int i = 0; i < 8; ++i) buf.push_back(static_cast<char>(v >> (8 * i)));
    };
    auto put_dec = [&](std::uint64_t v) {
        char t[24];
        int n = 0;
        do {
            t[n++] = static_cast<char>('0' + v % 10);
            v /= 10;
        } while (v);
        while (n) buf.push_back(t[--n]);
    };
    if (binary) {
        put_le(rows), put_le(cols), put_le(p);
        for (std::uint64_t i = 0; i < rows * cols; ++i) {
            put_le(data[i]);
            if (buf.size() >= (1u << 20)) flush();
        }
    } else {
        put_dec(rows), buf.push_back(' '), put_dec(cols), buf.push_back(' '), put_dec(p);
        buf.push_back('\n');
        for (std::uint64_t i = 0; i < rows; ++i) {
            for (std::uint64_t j = 0; j < cols; ++j) {
                if (j) buf.push_back(' ');
                put_dec(data[i * cols + j]);
            }
            buf.push_back('\n');
            if (buf.size() >= (1u << 20)) flush();
        }
    }
    flush();
}

}  // namespace wm
