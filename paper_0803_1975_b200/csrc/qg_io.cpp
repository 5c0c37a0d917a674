// qg_io.cpp — the reference's matrix file format (matrix_io.hpp:14-77) behind
// the C ABI: plain text
//
//     M <p> <rows> <cols>
//     <row-major residues, whitespace separated>
//
// read with the same stream-extraction rules and the same error texts, so a
// file either library accepts the other accepts, and a rejected file reports
// the same reason (ParseError, errors.hpp). Host-side parsing only: this is the
// data format on the input/output side of the GPU path, not part of it.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "../../include/qgemm_b200.h"
#include "qg_internal.h"

namespace {

// read_matrix, matrix_io.hpp:27-52. Returns QG_OK or QG_PARSE_ERROR (message
// in qg_last_error()).
int parse(std::istream& in, uint32_t* p_out, size_t* rows_out, size_t* cols_out, uint32_t** data_out) {
  std::string magic;
  if (!(in >> magic) || magic != "M") return qg::fail(QG_PARSE_ERROR, "matrix file must start with 'M <p> <rows> <cols>'");
  long long p = 0, rows = -1, cols = -1;
  if (!(in >> p >> rows >> cols) || p < 2 || rows < 0 || cols < 0) return qg::fail(QG_PARSE_ERROR, "bad matrix header");
  const size_t count = (size_t)rows * (size_t)cols;
  uint32_t* data = (uint32_t*)std::malloc((count ? count : 1) * sizeof(uint32_t));
  if (!data) return qg::fail(QG_INVALID_ARGUMENT, "out of host memory");
  for (size_t i = 0; i < count; ++i) {
    long long v;
    if (!(in >> v)) {
      std::free(data);
      return qg::fail(QG_PARSE_ERROR, "expected " + std::to_string(count) + " values, got " + std::to_string(i));
    }
    if (v < 0 || v >= p) {
      std::free(data);
      return qg::fail(QG_PARSE_ERROR, "value " + std::to_string(v) + " out of range [0, " + std::to_string(p - 1) + "]");
    }
    data[i] = (uint32_t)v;
  }
  long long extra;
  if (in >> extra) {
    std::free(data);
    return qg::fail(QG_PARSE_ERROR, "trailing values after " + std::to_string(count) + " entries");
  }
  *p_out = (uint32_t)p;  // truncated like static_cast<std::uint32_t>(p), matrix_io.hpp:36
  *rows_out = (size_t)rows;
  *cols_out = (size_t)cols;
  *data_out = data;
  return QG_OK;
}

}  // namespace

extern "C" {

int qg_parse_matrix(const char* text, size_t len, uint32_t* p, size_t* rows, size_t* cols, uint32_t** data) {
  if (!text || !p || !rows || !cols || !data) return QG_INVALID_ARGUMENT;
  std::istringstream in(std::string(text, len));
  return parse(in, p, rows, cols, data);
}

// read_matrix_file, matrix_io.hpp:54-62: errors are prefixed with the path.
int qg_read_matrix_file(const char* path, uint32_t* p, size_t* rows, size_t* cols, uint32_t** data) {
  if (!path || !p || !rows || !cols || !data) return QG_INVALID_ARGUMENT;
  std::ifstream in(path);
  if (!in) return qg::fail(QG_PARSE_ERROR, std::string("cannot open ") + path);
  const int st = parse(in, p, rows, cols, data);
  if (st == QG_PARSE_ERROR) return qg::fail(st, std::string(path) + ": " + qg_last_error());
  return st;
}

// write_matrix / write_matrix_file, matrix_io.hpp:64-75.
int qg_write_matrix_file(const char* path, uint32_t p, const uint32_t* data, size_t rows, size_t cols) {
  if (!path || (!data && rows * cols)) return QG_INVALID_ARGUMENT;
  std::ofstream out(path);
  if (!out) return qg::fail(QG_PARSE_ERROR, std::string("cannot open ") + path + " for writing");
  out << "M " << p << ' ' << rows << ' ' << cols << '\n';
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < cols; ++j) out << data[i * cols + j] << (j + 1 == cols ? '\n' : ' ');
  out.flush();
  if (!out) return qg::fail(QG_PARSE_ERROR, std::string("cannot write ") + path);
  return QG_OK;
}

void qg_free(void* ptr) { std::free(ptr); }

}  // extern "C"
