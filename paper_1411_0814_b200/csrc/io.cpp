// io.cpp -- host loader path for masked matrices (SURVEY.md section 8(f)
// row 1): the reference's NaN-CSV format and its dataset checksum
// (src/io.cpp:56-154 of /root/reference/proj, include/rsm/io.hpp:12-22).
//
//   load: one row per line, ',' separated; '\r' before '\n' dropped; a final
//         empty line ignored; each cell trimmed of isspace; an empty cell or
//         a case-insensitive "nan" (exactly three characters) is a hidden
//         entry; anything else must parse completely with strtod to a finite
//         value. Errors (errc::parse_io): "cannot open file: P",
//         "non-numeric token 'T' in P", "ragged row K in P" (K 1-based),
//         "empty matrix in P".
//   save: hidden cells as "NaN", observed ones "%.17g" (bit-lossless), '\n'
//         after every row; an empty matrix is errc::invalid_config.
//   checksum: FNV-1a 64 over the dims (two little-endian u64), then per cell
//         in row-major order one byte known?1:0 and, when known, the value's
//         8 IEEE bytes.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/rsm_b200.h"
#include "rsm_internal.h"

namespace {

struct IoError {
  rsm_status code;
  std::string msg;
};

[[noreturn]] void io_fail(rsm_status code, const std::string& msg) { throw IoError{code, msg}; }

template <class F>
rsm_status io_guard(F&& f) {
  try {
    f();
    return RSM_OK;
  } catch (const IoError& e) {
    rsmk::set_host_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    rsmk::set_host_error(e.what());
    return RSM_ERR_INTERNAL;
  }
}

bool is_nan_token(const char* b, size_t len) {
  return len == 3 && std::tolower((unsigned char)b[0]) == 'n' && std::tolower((unsigned char)b[1]) == 'a' &&
         std::tolower((unsigned char)b[2]) == 'n';
}

}  // namespace

extern "C" {

rsm_status rsm_load_matrix_csv(const char* path, double** values, uint8_t** mask, int64_t* m, int64_t* n) {
  return io_guard([&] {
    if (!path || !values || !mask || !m || !n) io_fail(RSM_ERR_INVALID_CONFIG, "null argument");
    const std::string p(path);
    std::ifstream in(p, std::ios::binary);
    if (!in) io_fail(RSM_ERR_PARSE_IO, "cannot open file: " + p);
    std::ostringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    std::vector<double> vals;
    std::vector<uint8_t> known;
    size_t width = 0, rows = 0;
    size_t pos = 0;
    const size_t N = text.size();
    std::string cell;
    while (pos < N) {
      size_t eol = text.find('\n', pos);
      const bool last = eol == std::string::npos;
      if (last) eol = N;
      size_t end = eol;
      if (end > pos && text[end - 1] == '\r') --end;
      // std::getline semantics: a final line without '\n' is still a line;
      // an empty line right before EOF is the trailing newline (io.cpp:64)
      if (end == pos && (last || eol + 1 >= N)) break;
      size_t cells = 0;
      size_t c0 = pos;
      for (;;) {
        size_t c1 = c0;
        while (c1 < end && text[c1] != ',') ++c1;
        size_t a = c0, b = c1;
        while (a < b && std::isspace((unsigned char)text[a])) ++a;
        while (b > a && std::isspace((unsigned char)text[b - 1])) --b;
        if (a == b || is_nan_token(text.data() + a, b - a)) {
          vals.push_back(0.0);
          known.push_back(0);
        } else {
          cell.assign(text, a, b - a);
          char* stop = nullptr;
          const double v = std::strtod(cell.c_str(), &stop);
          if (stop != cell.c_str() + cell.size() || !std::isfinite(v))
            io_fail(RSM_ERR_PARSE_IO, "non-numeric token '" + cell + "' in " + p);
          vals.push_back(v);
          known.push_back(1);
        }
        ++cells;
        if (c1 >= end) break;
        c0 = c1 + 1;
      }
      if (width == 0) width = cells;
      if (cells != width) io_fail(RSM_ERR_PARSE_IO, "ragged row " + std::to_string(rows + 1) + " in " + p);
      ++rows;
      if (last) break;
      pos = eol + 1;
    }
    if (rows == 0 || width == 0) io_fail(RSM_ERR_PARSE_IO, "empty matrix in " + p);
    double* V = (double*)std::malloc(sizeof(double) * rows * width);
    uint8_t* W = (uint8_t*)std::malloc(rows * width);
    if (!V || !W) {
      std::free(V);
      std::free(W);
      io_fail(RSM_ERR_INTERNAL, "out of host memory");
    }
    for (size_t q = 0; q < rows * width; ++q) {
      W[q] = known[q];
      V[q] = known[q] ? vals[q] : std::nan("");
    }
    *values = V;
    *mask = W;
    *m = (int64_t)rows;
    *n = (int64_t)width;
  });
}

rsm_status rsm_save_matrix_csv(const char* path, const double* values, const uint8_t* mask, int64_t m, int64_t n) {
  return io_guard([&] {
    if (m < 1 || n < 1) io_fail(RSM_ERR_INVALID_CONFIG, "cannot save an empty matrix");
    if (!path || !values || !mask) io_fail(RSM_ERR_INVALID_CONFIG, "null argument");
    std::string out;
    out.reserve((size_t)(m * n) * 8);
    char buf[40];
    for (int64_t i = 0; i < m; ++i) {
      for (int64_t j = 0; j < n; ++j) {
        if (j) out += ',';
        if (mask[i * n + j]) {
          std::snprintf(buf, sizeof buf, "%.17g", values[i * n + j]);
          out += buf;
        } else {
          out += "NaN";
        }
      }
      out += '\n';
    }
    const std::string p(path);
    std::ofstream f(p, std::ios::binary);
    if (!f) io_fail(RSM_ERR_PARSE_IO, "cannot open file for writing: " + p);
    f << out;
    if (!f) io_fail(RSM_ERR_PARSE_IO, "write failed: " + p);
  });
}

rsm_status rsm_dataset_checksum(const double* values, const uint8_t* mask, int64_t m, int64_t n, uint64_t* out) {
  return io_guard([&] {
    if (!out || m < 0 || n < 0 || (m * n > 0 && (!values || !mask))) io_fail(RSM_ERR_INVALID_CONFIG, "bad arguments");
    uint64_t h = 0xcbf29ce484222325ull;
    auto fnv = [&](const void* d, size_t len) {
      const unsigned char* q = (const unsigned char*)d;
      for (size_t k = 0; k < len; ++k) {
        h ^= q[k];
        h *= 0x100000001b3ull;
      }
    };
    const uint64_t dims[2] = {(uint64_t)m, (uint64_t)n};
    fnv(dims, sizeof dims);
    for (int64_t q = 0; q < m * n; ++q) {
      const unsigned char k = mask[q] ? 1 : 0;
      fnv(&k, 1);
      if (k) {
        uint64_t bits;
        std::memcpy(&bits, values + q, 8);
        fnv(&bits, 8);
      }
    }
    *out = h;
  });
}

void rsm_free(void* p) { std::free(p); }

}  // extern "C"
