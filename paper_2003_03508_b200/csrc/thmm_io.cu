// thmm_io.cu -- observation CSV ingestion straight to the arrays the device
// stream takes (host code; compiled with the rest of libthmm).
//
// Format and error behaviour of reference dataio.load_dataset
// (dataio.py:46-87): header `timestamp,lon,lat`; one record per row; a quiet
// hour leaves both coordinate fields empty; ISO-8601 timestamps strictly
// increasing; every malformed row is reported with its line number.  The
// reference builds one Python Observation per row; here a single pass fills
// present/lon/lat (and optionally the timestamps as microseconds).
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "thmm.h"

namespace {

void io_err(char* err, size_t errlen, const char* fmt, ...) {
  if (!err || errlen == 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r' || s[a] == '\n')) ++a;
  while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r' || s[b - 1] == '\n')) --b;
  return s.substr(a, b - a);
}

// Split one CSV row on commas (the reference writer never quotes these fields;
// a quoted field is unquoted with "" -> ").
std::vector<std::string> split_row(const std::string& line) {
  std::vector<std::string> out;
  std::string cur;
  bool quoted = false;
  for (size_t i = 0; i < line.size(); ++i) {
    const char c = line[i];
    if (quoted) {
      if (c == '"' && i + 1 < line.size() && line[i + 1] == '"') {
        cur.push_back('"');
        ++i;
      } else if (c == '"') {
        quoted = false;
      } else {
        cur.push_back(c);
      }
    } else if (c == '"' && strip(cur).empty()) {
      quoted = true;
    } else if (c == ',') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  out.push_back(cur);
  return out;
}

bool digits(const std::string& s, size_t pos, size_t n, int& v) {
  if (pos + n > s.size()) return false;
  v = 0;
  for (size_t i = 0; i < n; ++i) {
    const char c = s[pos + i];
    if (c < '0' || c > '9') return false;
    v = v * 10 + (c - '0');
  }
  return true;
}

int64_t days_from_civil(int64_t y, unsigned m, unsigned d) {  // proleptic Gregorian
  y -= m <= 2;
  const int64_t era = (y >= 0 ? y : y - 399) / 400;
  const unsigned yoe = static_cast<unsigned>(y - era * 400);
  const unsigned doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
  const unsigned doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + static_cast<int64_t>(doe) - 719468;
}

// ISO-8601 subset accepted by datetime.fromisoformat:
// YYYY-MM-DD[(T| )HH[:MM[:SS[.f{1,6}]]][Z|(+|-)HH:MM[:SS]]] -> microseconds.
bool parse_iso(const std::string& s, int64_t& us) {
  int y, mo, d;
  if (!digits(s, 0, 4, y) || s.size() < 10 || s[4] != '-' || !digits(s, 5, 2, mo) || s[7] != '-' ||
      !digits(s, 8, 2, d))
    return false;
  static const int mdays[] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  const bool leap = (y % 4 == 0 && y % 100 != 0) || y % 400 == 0;
  if (mo < 1 || mo > 12 || d < 1 || d > mdays[mo - 1] + (mo == 2 && leap ? 1 : 0) || y < 1) return false;
  int h = 0, mi = 0, se = 0;
  int64_t frac = 0;
  size_t p = 10;
  if (p < s.size()) {
    if (s[p] != 'T' && s[p] != ' ') return false;
    ++p;
    if (!digits(s, p, 2, h)) return false;
    p += 2;
    if (p < s.size() && s[p] == ':') {
      if (!digits(s, p + 1, 2, mi)) return false;
      p += 3;
      if (p < s.size() && s[p] == ':') {
        if (!digits(s, p + 1, 2, se)) return false;
        p += 3;
        if (p < s.size() && (s[p] == '.' || s[p] == ',')) {
          ++p;
          int nd = 0;  // any number of digits; beyond microseconds they are truncated
          while (p < s.size() && s[p] >= '0' && s[p] <= '9') {
            if (nd < 6) frac = frac * 10 + (s[p] - '0');
            ++p;
            ++nd;
          }
          if (nd == 0) return false;
          for (; nd < 6; ++nd) frac *= 10;
        }
      }
    }
    if (h > 23 || mi > 59 || se > 59) return false;
    int64_t off = 0;
    if (p < s.size()) {
      if (s[p] == 'Z' && p + 1 == s.size()) {
        ++p;
      } else if (s[p] == '+' || s[p] == '-') {
        const int sign = s[p] == '-' ? -1 : 1;
        int oh, om = 0, os = 0;
        if (!digits(s, p + 1, 2, oh)) return false;
        p += 3;
        if (p < s.size() && s[p] == ':') {
          if (!digits(s, p + 1, 2, om)) return false;
          p += 3;
          if (p < s.size() && s[p] == ':') {
            if (!digits(s, p + 1, 2, os)) return false;
            p += 3;
          }
        }
        off = sign * (oh * 3600LL + om * 60LL + os);
      } else {
        return false;
      }
    }
    if (p != s.size()) return false;
    us = ((days_from_civil(y, mo, d) * 86400LL + h * 3600LL + mi * 60LL + se - off) * 1000000LL) + frac;
    return true;
  }
  us = days_from_civil(y, mo, d) * 86400LL * 1000000LL;
  return true;
}

bool parse_float(const std::string& s, double& v) {
  if (s.empty()) return false;
  if (s.size() > 1 && s[0] == '0' && (s[1] == 'x' || s[1] == 'X')) return false;  // float() rejects hex
  errno = 0;
  char* end = nullptr;
  v = std::strtod(s.c_str(), &end);
  return end == s.c_str() + s.size();
}

// One pass over the file; when `present` is non-null the arrays are filled
// (capacity n).  Returns the record count through *count.
int scan(const char* path, int64_t n, uint8_t* present, double* lon, double* lat, int64_t* t_us, int64_t* count,
         char* err, size_t errlen) {
  FILE* fh = std::fopen(path, "rb");
  if (!fh) {
    io_err(err, errlen, "cannot open %s", path);
    return THMM_EINVAL;
  }
  std::string line;
  std::vector<char> buf(1 << 16);
  int64_t lineno = 0, rec = 0, prev = 0;
  bool have_prev = false, header = false;
  int rc = THMM_OK;
  auto next_line = [&](std::string& out) -> bool {
    out.clear();
    int c;
    bool any = false;
    while ((c = std::fgetc(fh)) != EOF) {
      any = true;
      if (c == '\n') return true;
      out.push_back(static_cast<char>(c));
    }
    return any;
  };
  while (rc == THMM_OK && next_line(line)) {
    ++lineno;
    if (!header) {
      const std::vector<std::string> h = split_row(line);
      if (h.size() != 3 || strip(h[0]) != "timestamp" || strip(h[1]) != "lon" || strip(h[2]) != "lat") {
        io_err(err, errlen, "line 1: header must be timestamp,lon,lat");
        rc = THMM_EINVAL;
        break;
      }
      header = true;
      continue;
    }
    if (line.empty() || (line.size() == 1 && line[0] == '\r')) continue;
    const std::vector<std::string> f = split_row(line);
    if (f.size() != 3) {
      io_err(err, errlen, "line %lld: expected 3 fields, got %d", static_cast<long long>(lineno),
             static_cast<int>(f.size()));
      rc = THMM_EINVAL;
      break;
    }
    const std::string ts = strip(f[0]), xs = strip(f[1]), ys = strip(f[2]);
    int64_t us = 0;
    if (!parse_iso(ts, us)) {
      io_err(err, errlen, "line %lld: bad timestamp '%s'", static_cast<long long>(lineno), ts.c_str());
      rc = THMM_EINVAL;
      break;
    }
    if (have_prev && us <= prev) {
      io_err(err, errlen, "line %lld: timestamps must be strictly increasing", static_cast<long long>(lineno));
      rc = THMM_EINVAL;
      break;
    }
    prev = us;
    have_prev = true;
    bool pres = false;
    double x = 0.0, y = 0.0;
    if (xs.empty() && ys.empty()) {
      pres = false;
    } else if (xs.empty() || ys.empty()) {
      io_err(err, errlen, "line %lld: lon and lat must be both present or both empty",
             static_cast<long long>(lineno));
      rc = THMM_EINVAL;
      break;
    } else {
      if (!parse_float(xs, x) || !parse_float(ys, y)) {
        io_err(err, errlen, "line %lld: bad coordinate", static_cast<long long>(lineno));
        rc = THMM_EINVAL;
        break;
      }
      if (!std::isfinite(x) || !std::isfinite(y)) {
        io_err(err, errlen, "line %lld: coordinates must be finite", static_cast<long long>(lineno));
        rc = THMM_EINVAL;
        break;
      }
      pres = true;
    }
    if (present) {
      if (rec >= n) {
        io_err(err, errlen, "file changed between count and read");
        rc = THMM_EINVAL;
        break;
      }
      present[rec] = pres ? 1 : 0;
      lon[rec] = pres ? x : 0.0;
      lat[rec] = pres ? y : 0.0;
      if (t_us) t_us[rec] = us;
    }
    ++rec;
  }
  if (rc == THMM_OK && !header) {
    io_err(err, errlen, "line 1: missing header");
    rc = THMM_EINVAL;
  }
  std::fclose(fh);
  *count = rec;
  return rc;
}

}  // namespace

extern "C" {

int thmm_csv_count(const char* path, int64_t* n, char* err, size_t errlen) {
  if (!path || !n) {
    io_err(err, errlen, "null argument");
    return THMM_EINVAL;
  }
  return scan(path, 0, nullptr, nullptr, nullptr, nullptr, n, err, errlen);
}

int thmm_csv_read(const char* path, int64_t n, uint8_t* present, double* lon, double* lat, int64_t* t_us,
                  char* err, size_t errlen) {
  if (!path || !present || !lon || !lat) {
    io_err(err, errlen, "null argument");
    return THMM_EINVAL;
  }
  int64_t count = 0;
  const int rc = scan(path, n, present, lon, lat, t_us, &count, err, errlen);
  if (rc == THMM_OK && count != n) {
    io_err(err, errlen, "file changed between count and read");
    return THMM_EINVAL;
  }
  return rc;
}

}  // extern "C"
