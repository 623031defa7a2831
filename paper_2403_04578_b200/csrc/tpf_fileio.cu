// Native load / voltage tables (host code only): the file formats around the
// hot path, which at C2 scale (525,600 rows x 200
// fields, ~2.3 GB of text) take far longer in the reference's Python loops
// than the GPU solve.
//
//   loads    fileio.py:196-234  header p_1,q_1,...,p_b,q_b; one row per case
//   voltages fileio.py:237-253  header vm_1,va_1,...,converged; "%.17g" cells
//
// Parsing is correctly rounded (strtod), like Python's float(); fields that
// strtod would read differently from float() (hex, underscores, overlong) are
// reported as TPF_ERR_UNSUPPORTED so the caller can use its exact Python
// reader.  Formatting is "%.17g" (correctly rounded, like Python's
// f"{x:.17g}"), with every NaN printed as "nan" as Python does.  Rows are
// parsed / formatted by a pool of threads over contiguous row ranges; output
// order is the row order, so files are byte-identical run to run.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <locale.h>
#include <string>
#include <thread>
#include <vector>

#include "tpf_internal.h"

namespace tpf {
namespace {

// Python's float() and f"{x:.17g}" ignore LC_NUMERIC; strtod/snprintf follow
// it.  Every parse and format here uses the "C" locale explicitly, so a
// process that called setlocale(LC_ALL, "") under a comma-decimal locale
// still reads and writes the reference's bytes.
locale_t c_locale() {
  static const locale_t loc = newlocale(LC_ALL_MASK, "C", locale_t(0));
  return loc;
}


bool read_file(const char* path, std::string& out) {
  FILE* f = fopen(path, "rb");
  if (!f) return false;
  if (fseek(f, 0, SEEK_END) != 0) {
    fclose(f);
    return false;
  }
  const long n = ftell(f);
  if (n < 0) {
    fclose(f);
    return false;
  }
  rewind(f);
  out.resize(size_t(n));
  const size_t got = n ? fread(&out[0], 1, size_t(n), f) : 0;
  fclose(f);
  return got == size_t(n);
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

// Line spans [begin, end) of the text, newline excluded; the last line may lack one.
void split_lines(const std::string& s, std::vector<std::pair<size_t, size_t>>& lines) {
  size_t p = 0;
  const size_t n = s.size();
  while (p < n) {
    const void* nl = memchr(s.data() + p, '\n', n - p);
    const size_t e = nl ? size_t(static_cast<const char*>(nl) - s.data()) : n;
    lines.emplace_back(p, e);
    p = e + 1;
  }
}

bool blank(const std::string& s, size_t b, size_t e) {
  for (size_t i = b; i < e; ++i)
    if (!is_ws(s[i])) return false;
  return true;
}

std::string load_header(int b) {
  std::string h;
  for (int i = 1; i <= b; ++i) {
    if (i > 1) h += ',';
    h += "p_" + std::to_string(i) + ",q_" + std::to_string(i);
  }
  return h;
}

// 0 ok, 1 not a number for Python float() either, 2 needs the exact Python reader
int parse_field(const char* b, const char* e, double* out) {
  while (b < e && is_ws(*b)) ++b;
  while (e > b && is_ws(e[-1])) --e;
  const size_t n = size_t(e - b);
  if (n == 0) return 1;
  if (n > 63) return 2;
  char buf[64];
  for (size_t i = 0; i < n; ++i) {
    const char c = b[i];
    const bool numeric = (c >= '0' && c <= '9') || c == '.' || c == '+' || c == '-' || c == 'e' || c == 'E';
    if (!numeric) return 2;  // inf/nan words, hex, underscores, garbage: the exact reader decides
    buf[i] = c;
  }
  buf[n] = '\0';
  char* end = nullptr;
  errno = 0;
  const double v = strtod_l(buf, &end, c_locale());
  if (end != buf + n) return 1;
  *out = v;  // overflow gives +-inf and underflow a denormal/0, as float() does
  return 0;
}

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" int tpf_loads_csv_scan(const char* path, int32_t* b_out, int64_t* tau_out) {
  if (!path || !b_out || !tau_out) return set_error(TPF_ERR_INVALID, "tpf_loads_csv_scan: null argument");
  std::string text;
  if (!read_file(path, text)) return set_error(TPF_ERR_INVALID, (std::string(path) + ": no such file").c_str());
  std::vector<std::pair<size_t, size_t>> lines;
  split_lines(text, lines);
  if (lines.empty() || blank(text, lines[0].first, lines[0].second))
    return set_error(TPF_ERR_INVALID, (std::string(path) + ": empty file").c_str());
  size_t hb = lines[0].first, he = lines[0].second;
  while (hb < he && is_ws(text[hb])) ++hb;
  while (he > hb && is_ws(text[he - 1])) --he;
  const std::string header = text.substr(hb, he - hb);
  int64_t commas = 0;
  for (char c : header) commas += c == ',';
  const int64_t names = commas + 1;
  if (names % 2 != 0)
    return set_error(TPF_ERR_INVALID, (std::string(path) + ": header must hold p_<node>,q_<node> pairs").c_str());
  const int b = int(names / 2);
  if (header != load_header(b))
    return set_error(TPF_ERR_INVALID,
                     (std::string(path) + ": header does not match the expected p_1,q_1,...,p_" + std::to_string(b) +
                      ",q_" + std::to_string(b) + " layout")
                         .c_str());
  int64_t tau = 0;
  for (size_t k = 1; k < lines.size(); ++k) tau += !blank(text, lines[k].first, lines[k].second);
  if (tau == 0) return set_error(TPF_ERR_INVALID, (std::string(path) + ": no load cases").c_str());
  *b_out = b;
  *tau_out = tau;
  return TPF_OK;
}

extern "C" int tpf_loads_csv_read(const char* path, int32_t b, int64_t tau, double* values, int64_t* bad_line,
                                  int32_t threads) {
  if (!path || b < 1 || tau < 1 || !values) return set_error(TPF_ERR_INVALID, "tpf_loads_csv_read: bad argument");
  std::string text;
  if (!read_file(path, text)) return set_error(TPF_ERR_INVALID, (std::string(path) + ": no such file").c_str());
  std::vector<std::pair<size_t, size_t>> lines;
  split_lines(text, lines);
  std::vector<int64_t> data;  // line index of every non-blank data line
  data.reserve(size_t(tau));
  for (size_t k = 1; k < lines.size(); ++k)
    if (!blank(text, lines[k].first, lines[k].second)) data.push_back(int64_t(k));
  if (int64_t(data.size()) != tau) return set_error(TPF_ERR_INVALID, "tpf_loads_csv_read: file changed since scan");
  int nt = threads > 0 ? threads : int(std::thread::hardware_concurrency());
  if (nt < 1) nt = 1;
  if (int64_t(nt) > tau) nt = int(tau);
  // per-thread first failure: (line index, code)
  std::vector<int64_t> fail_line(static_cast<size_t>(nt), -1);
  std::vector<int> fail_code(static_cast<size_t>(nt), 0);
  auto work = [&](int w) {
    const int64_t lo = tau * w / nt, hi = tau * (w + 1) / nt;
    for (int64_t j = lo; j < hi; ++j) {
      const auto& ln = lines[size_t(data[size_t(j)])];
      const char* p = text.data() + ln.first;
      const char* end = text.data() + ln.second;
      // strip(), then exactly 2b comma-separated fields
      while (p < end && is_ws(*p)) ++p;
      while (end > p && is_ws(end[-1])) --end;
      int64_t commas = 0;
      for (const char* q = p; q < end; ++q) commas += *q == ',';
      if (commas + 1 != 2 * int64_t(b)) {
        fail_line[size_t(w)] = data[size_t(j)];
        fail_code[size_t(w)] = 1;
        return;
      }
      const char* f = p;
      for (int k = 0; k < 2 * b; ++k) {
        const char* c = static_cast<const char*>(memchr(f, ',', size_t(end - f)));
        if (!c) c = end;
        double v = 0.0;
        const int rc = parse_field(f, c, &v);
        if (rc != 0) {
          fail_line[size_t(w)] = data[size_t(j)];
          fail_code[size_t(w)] = rc;
          return;
        }
        values[2 * (int64_t(k / 2) * tau + j) + (k & 1)] = v;  // node k/2, case j: (p, q)
        f = c + 1;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < nt; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& t : pool) t.join();
  for (int w = 0; w < nt; ++w) {
    if (fail_line[size_t(w)] >= 0) {  // earliest failing line (thread ranges are ordered)
      if (bad_line) *bad_line = fail_line[size_t(w)] + 1;  // 1-based line number
      return fail_code[size_t(w)] == 2
                 ? set_error(TPF_ERR_UNSUPPORTED, "field needs the exact Python float() reader")
                 : set_error(TPF_ERR_INVALID, "malformed line");
    }
  }
  return TPF_OK;
}

extern "C" int tpf_write_pairs_csv(const char* path, const char* header, int32_t b, int64_t tau, const double* x,
                                   const double* y, int64_t node_stride, int64_t case_stride, const uint8_t* flag,
                                   int32_t threads) {
  if (!path || !header || b < 1 || tau < 0 || !x || !y)
    return set_error(TPF_ERR_INVALID, "tpf_write_pairs_csv: bad argument");
  FILE* f = fopen(path, "wb");
  if (!f) return set_error(TPF_ERR_INVALID, (std::string(path) + ": cannot open for writing").c_str());
  bool ok = fputs(header, f) >= 0 && fputc('\n', f) != EOF;
  int nt = threads > 0 ? threads : int(std::thread::hardware_concurrency());
  if (nt < 1) nt = 1;
  // rows per formatting task (blocks are written in order): all threads busy,
  // at most 4096 rows buffered per thread
  int64_t block = (tau + nt - 1) / (nt > 0 ? nt : 1);
  if (block > 4096) block = 4096;
  if (block < 64) block = 64;
  std::vector<std::string> out(static_cast<size_t>(nt));
  auto fmt = [](std::string& s, double v) {
    char buf[40];
    if (std::isnan(v)) {
      s += "nan";
      return;
    }
    const int n = snprintf(buf, sizeof buf, "%.17g", v);
    s.append(buf, size_t(n));
  };
  for (int64_t r0 = 0; ok && r0 < tau; r0 += block * nt) {
    auto work = [&](int w) {
      const locale_t prev = uselocale(c_locale());  // this thread only
      std::string& s = out[size_t(w)];
      s.clear();
      const int64_t lo = r0 + block * w, hi = std::min(tau, lo + block);
      for (int64_t j = lo; j < hi; ++j) {
        for (int i = 0; i < b; ++i) {
          const int64_t at = int64_t(i) * node_stride + j * case_stride;
          if (i) s += ',';
          fmt(s, x[at]);
          s += ',';
          fmt(s, y[at]);
        }
        if (flag) s += flag[j] ? ",1" : ",0";
        s += '\n';
      }
      uselocale(prev);
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < nt; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    for (int w = 0; w < nt && ok; ++w) ok = fwrite(out[size_t(w)].data(), 1, out[size_t(w)].size(), f) == out[size_t(w)].size();
  }
  ok = (fclose(f) == 0) && ok;
  if (!ok) return set_error(TPF_ERR_INVALID, (std::string(path) + ": write failed").c_str());
  return TPF_OK;
}
