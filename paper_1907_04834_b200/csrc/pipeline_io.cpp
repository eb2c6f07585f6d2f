// pipeline_io.cpp -- point-cloud file formats on either side of the hot path
// (SURVEY.md §8f rank 3): whitespace "x y z" text and legacy-VTK ASCII
// polydata, with the reference's reading rules and error classes
// (proj/src/pipeline_io.cpp:23-149) and its %.17g output, so every double
// survives a write/read round trip bit for bit. Host-only by nature (text
// parsing); the points it produces feed the device C ABI unchanged.
#include <cerrno>
#include <cmath>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "geoshoot_b200.h"

namespace {

thread_local long long g_parse_line = 0;
thread_local std::string g_io_msg;

gs_status parse_error(long long line, const std::string& what) {
  g_parse_line = line;
  g_io_msg = "line " + std::to_string(line) + ": " + what;
  return GS_PARSE_ERROR;
}

gs_status unsupported(const std::string& what) {
  g_io_msg = what;
  return GS_UNSUPPORTED_FORMAT;
}

std::string trimmed(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace((unsigned char)s[b])) ++b;
  while (e > b && std::isspace((unsigned char)s[e - 1])) --e;
  return s.substr(b, e - b);
}

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
    const size_t b = i;
    while (i < s.size() && !std::isspace((unsigned char)s[i])) ++i;
    if (i > b) out.push_back(s.substr(b, i - b));
  }
  return out;
}

// Stream-extraction number syntax (digits, sign, point, exponent; no inf/nan
// or hex), overflow rejected -- what `istream >> double` accepts for xyz text.
bool stream_number(const std::string& tok, double& v) {
  for (char c : tok)
    if (!(std::isdigit((unsigned char)c) || c == '+' || c == '-' || c == '.' || c == 'e' || c == 'E'))
      return false;
  errno = 0;
  char* end = nullptr;
  v = std::strtod(tok.c_str(), &end);
  if (end != tok.c_str() + tok.size() || tok.empty()) return false;
  if (errno == ERANGE && (v == HUGE_VAL || v == -HUGE_VAL)) return false;
  return true;
}

// Full strtod syntax (std::stod), whole token consumed -- the VTK reader's rule.
bool full_number(const std::string& tok, double& v) {
  errno = 0;
  char* end = nullptr;
  v = std::strtod(tok.c_str(), &end);
  if (tok.empty() || end != tok.c_str() + tok.size()) return false;
  if (errno == ERANGE && (v == HUGE_VAL || v == -HUGE_VAL)) return false;  // std::stod throws
  return true;
}

gs_status read_xyz(std::istream& in, std::vector<double>& out) {
  std::string line;
  long long lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const std::string body = trimmed(line);
    if (body.empty() || body[0] == '#') continue;
    const std::vector<std::string> tok = split_ws(body);
    double v[3];
    for (int a = 0; a < 3; ++a)
      if ((size_t)a >= tok.size() || !stream_number(tok[a], v[a]))
        return parse_error(lineno, "expected three coordinates");
    if (tok.size() > 3) return parse_error(lineno, "trailing content: " + tok[3]);
    out.insert(out.end(), v, v + 3);
  }
  if (out.empty()) return parse_error(lineno, "no points");
  return GS_OK;
}

gs_status read_vtk(std::istream& in, std::vector<double>& out) {
  std::vector<std::string> lines;
  std::string line;
  while (std::getline(in, line)) lines.push_back(line);
  if (lines.empty() || lines[0].rfind("# vtk DataFile Version", 0) != 0)
    return unsupported("not a legacy vtk data file");
  if (lines.size() < 4) return parse_error((long long)lines.size(), "truncated header");
  if (trimmed(lines[2]) != "ASCII")
    return unsupported("only ASCII vtk files are supported, got '" + trimmed(lines[2]) + "'");
  if (trimmed(lines[3]) != "DATASET POLYDATA") return unsupported("only DATASET POLYDATA is supported");
  // token stream from line 5 on, remembering each token's 1-based line
  std::vector<std::pair<std::string, long long>> toks;
  for (size_t l = 4; l < lines.size(); ++l)
    for (auto& t : split_ws(lines[l])) toks.emplace_back(t, (long long)l + 1);
  const long long end_line = (long long)lines.size() + 1;
  size_t k = 0;
  while (k < toks.size() && toks[k].first != "POINTS") ++k;
  if (k == toks.size()) return parse_error(end_line, "no POINTS section");
  ++k;
  auto next_num = [&](double& v) -> gs_status {
    if (k >= toks.size()) return parse_error(end_line, "unexpected end of file");
    const auto& t = toks[k++];
    if (!full_number(t.first, v)) return parse_error(t.second, "expected a number, got '" + t.first + "'");
    return GS_OK;
  };
  double nraw = 0;
  gs_status st = next_num(nraw);
  if (st != GS_OK) return st;
  const long long count_line = toks[k - 1].second;
  const long long n = (long long)nraw;
  if (!(nraw > 0) || (double)n != nraw) return parse_error(count_line, "bad POINTS count");
  if (k >= toks.size() || (toks[k].first != "float" && toks[k].first != "double"))
    return parse_error(k < toks.size() ? toks[k].second : end_line, "POINTS type must be float or double");
  ++k;
  out.reserve(3 * (size_t)n);
  for (long long i = 0; i < 3 * n; ++i) {
    double v = 0;
    if ((st = next_num(v)) != GS_OK) return st;
    out.push_back(v);
  }
  return GS_OK;  // cells (VERTICES / POLYGONS / ...) are ignored
}

void put_row(std::ostream& os, const double* p) {
  char buf[96];
  std::snprintf(buf, sizeof buf, "%.17g %.17g %.17g\n", p[0], p[1], p[2]);
  os << buf;
}

}  // namespace

extern "C" {

int32_t gs_format_for_path(const char* path) {
  const char* dot = path ? std::strrchr(path, '.') : nullptr;
  return (dot && std::strcmp(dot, ".vtk") == 0) ? GS_FORMAT_VTK : GS_FORMAT_XYZ;
}

long long gs_last_parse_line(void) { return g_parse_line; }
const char* gs_last_io_error(void) { return g_io_msg.c_str(); }

gs_status gs_read_points(const char* path, int32_t format, double* xyz_out, int64_t capacity,
                         int64_t* n_out) {
  if (!path || !n_out) return GS_INVALID_ARGUMENT;
  std::ifstream in(path);
  if (!in) {
    g_io_msg = std::string("cannot open '") + path + "' for reading";
    return GS_IO_ERROR;
  }
  std::vector<double> v;
  const gs_status st = format == GS_FORMAT_VTK ? read_vtk(in, v) : read_xyz(in, v);
  if (st != GS_OK) return st;
  for (double x : v)
    if (!std::isfinite(x)) {  // PointSet constructor (core.hpp:126-131)
      g_io_msg = "PointSet: non-finite coordinate";
      return GS_INVALID_ARGUMENT;
    }
  *n_out = (int64_t)(v.size() / 3);
  if (xyz_out) {
    if (capacity < *n_out) return GS_DIMENSION_MISMATCH;
    std::memcpy(xyz_out, v.data(), sizeof(double) * v.size());
  }
  return GS_OK;
}

gs_status gs_write_points(const char* path, int32_t format, int64_t n, const double* xyz,
                          const char* const* header, int32_t n_header) {
  if (!path || (!xyz && n > 0)) return GS_INVALID_ARGUMENT;
  std::ofstream os(path);
  if (!os) {
    g_io_msg = std::string("cannot open '") + path + "' for writing";
    return GS_IO_ERROR;
  }
  if (format == GS_FORMAT_VTK) {
    os << "# vtk DataFile Version 3.0\n";
    os << (n_header > 0 && header ? header[0] : "point set") << '\n';
    os << "ASCII\nDATASET POLYDATA\n";
    os << "POINTS " << n << " double\n";
    for (int64_t i = 0; i < n; ++i) put_row(os, xyz + 3 * i);
    os << "VERTICES " << n << ' ' << 2 * n << '\n';
    for (int64_t i = 0; i < n; ++i) os << "1 " << i << '\n';
  } else {
    for (int32_t h = 0; h < n_header && header; ++h) os << "# " << header[h] << '\n';
    for (int64_t i = 0; i < n; ++i) put_row(os, xyz + 3 * i);
  }
  return os ? GS_OK : GS_IO_ERROR;
}

}  // extern "C"
