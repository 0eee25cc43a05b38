// egs_arena_io.cpp — arena input/output for the solve path (SURVEY.md §8f
// next #1): the reference's text format and a binary format that loads
// without parsing.
//
//   egs_host_arena_build   GameArena::build (proj/src/arena.cpp:17-78):
//                          validation, stable counting sort by source,
//                          compute_stats (arena.cpp:80-108)
//   egs_arena_parse_text   parse_arena (proj/src/io.cpp:87-149) + build, on
//                          every host thread: the reference's records,
//                          checks and error kinds, reported for the first
//                          offending line as the reference reports it
//   egs_arena_write_text   write_arena (io.cpp:151-176), byte-identical
//   egs_arena_save/_load   the binary format (below): the CSR spans with
//                          the weights narrowed to the narrowest of
//                          int8/16/32/64 holding max |w|; loading is one
//                          read per span plus validation, no parsing
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "egs_gpu.h"
#include "egs_host_arena.h"

void egs_internal_set_error(const std::string& msg);

namespace {

unsigned host_threads() { return std::max(1u, std::min(32u, std::thread::hardware_concurrency())); }

template <class Fn>
void run_threads(unsigned T, Fn&& fn) {
  if (T <= 1) {
    fn(0u);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < T; ++t) pool.emplace_back([&fn, t] { fn(t); });
  for (auto& th : pool) th.join();
}

// An input error of the reference's loader (errors.hpp): kind + message as
// the reference formats it.
struct InputError {
  bool set = false;
  uint64_t line = 0;  // order key: the first error in file order wins
  std::string msg;
  int code = EGS_ERR_INPUT;
  void raise(uint64_t at, std::string m, int c = EGS_ERR_INPUT) {
    if (!set || at < line) {
      set = true;
      line = at;
      msg = std::move(m);
      code = c;
    }
  }
};

int fail(const InputError& e) {
  egs_internal_set_error(e.msg);
  return e.code;
}

// ---------------------------------------------------------------- build ----
// GameArena::build: owners cover every vertex, ids in range, no INT64_MIN
// weight, every vertex has a successor, rows keep input order.
int build_arena(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                const int64_t* w, const uint8_t* owners, bool pinned, egs_host_arena** out) {
  InputError err;
  for (uint64_t i = 0; i < m; ++i) {
    if (src[i] >= n) {
      err.raise(0, "DanglingVertexIdError: edge references unknown vertex id " +
                       std::to_string(src[i]));
      break;
    }
    if (dst[i] >= n) {
      err.raise(0, "DanglingVertexIdError: edge references unknown vertex id " +
                       std::to_string(dst[i]));
      break;
    }
    if (w[i] == std::numeric_limits<int64_t>::min()) {
      err.raise(0, "edge weight magnitude not representable", EGS_ERR_UNSUPPORTED);
      break;
    }
  }
  if (err.set) return fail(err);
  egs_host_arena* a = egs_internal_arena_alloc(n, m, pinned);
  if (!a) {
    egs_internal_set_error("host allocation failed");
    return EGS_ERR_CUDA;
  }
  for (uint32_t v = 0; v < n; ++v) a->owner[v] = owners[v] ? 1 : 0;
  // rows: already grouped by ascending source (write_arena's order)?  Then
  // the CSR is the input itself; else the reference's stable counting sort.
  bool sorted = true;
  for (uint64_t i = 1; i < m && sorted; ++i) sorted = src[i - 1] <= src[i];
  std::fill(a->off, a->off + (size_t)n + 1, 0ull);
  for (uint64_t i = 0; i < m; ++i) a->off[src[i] + 1]++;
  for (uint32_t v = 0; v < n; ++v) {
    if (a->off[v + 1] == 0) {
      egs_internal_arena_free(a);
      egs_internal_set_error("NonTotalArenaError: vertex " + std::to_string(v) +
                             " has no outgoing edge");
      return EGS_ERR_INPUT;
    }
    a->off[v + 1] += a->off[v];
  }
  if (sorted) {
    std::memcpy(a->dst, dst, m * sizeof(uint32_t));
    std::memcpy(a->w, w, m * sizeof(int64_t));
  } else {
    std::vector<uint64_t> cursor(a->off, a->off + n);
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t slot = cursor[src[i]]++;
      a->dst[slot] = dst[i];
      a->w[slot] = w[i];
    }
  }
  const int rc = egs_internal_finish_stats(a);
  if (rc != EGS_OK) {
    egs_internal_arena_free(a);
    return rc;
  }
  *out = a;
  return EGS_OK;
}

// ----------------------------------------------------------------- text ----
// parse_arena's records: "eg <V> <E>", then V lines "v <id> <owner>" with
// ids 0..V-1 in order, then E lines "e <src> <dst> <weight>"; blank lines
// and lines starting with '#' are skipped; a trailing '\r' is dropped;
// fields are separated by single spaces (io.cpp:29-83, 87-149).
struct Fields {
  std::string_view f[5];
  int count = 0;
  bool empty_field = false;
};

Fields split(std::string_view line) {
  Fields out;
  size_t start = 0;
  while (true) {
    const size_t sp = line.find(' ', start);
    const std::string_view piece =
        sp == std::string_view::npos ? line.substr(start) : line.substr(start, sp - start);
    if (out.count < 5) out.f[out.count] = piece;
    ++out.count;
    if (piece.empty()) out.empty_field = true;
    if (sp == std::string_view::npos) break;
    start = sp + 1;
  }
  return out;
}

template <class T>
bool number(std::string_view s, T& v) {
  auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  return r.ec == std::errc() && r.ptr == s.data() + s.size();
}

// Iterates the records (non-blank, non-comment lines) of text[lo, hi),
// which starts at a line boundary; `line` is the 1-based line number.
template <class Fn>
void for_records(const char* text, size_t lo, size_t hi, uint64_t first_line, Fn&& fn) {
  uint64_t line_no = first_line;
  size_t pos = lo;
  while (pos < hi) {
    const char* nl = static_cast<const char*>(std::memchr(text + pos, '\n', hi - pos));
    const size_t end = nl ? (size_t)(nl - text) : hi;
    std::string_view raw(text + pos, end - pos);
    pos = nl ? end + 1 : hi;
    ++line_no;
    if (!raw.empty() && raw.back() == '\r') raw.remove_suffix(1);
    if (raw.empty() || raw.front() == '#') continue;
    if (!fn(raw, line_no)) return;
  }
}

int parse_text(const char* text, size_t len, bool pinned, egs_host_arena** out) {
  InputError err;
  // header: the first record
  size_t pos = 0;
  uint64_t line_no = 0;
  std::string_view header;
  bool have = false;
  while (pos < len && !have) {
    const char* nl = static_cast<const char*>(std::memchr(text + pos, '\n', len - pos));
    const size_t end = nl ? (size_t)(nl - text) : len;
    std::string_view raw(text + pos, end - pos);
    pos = nl ? end + 1 : len;
    ++line_no;
    if (!raw.empty() && raw.back() == '\r') raw.remove_suffix(1);
    if (raw.empty() || raw.front() == '#') continue;
    header = raw;
    have = true;
  }
  if (!have) {
    err.raise(1, "SyntaxError: line 1: missing 'eg <vertices> <edges>' header");
    return fail(err);
  }
  {
    const Fields h = split(header);
    auto syntax = [&](const std::string& why) {
      err.raise(line_no, "SyntaxError: line " + std::to_string(line_no) + ": " + why);
    };
    if (h.empty_field) syntax("fields must be separated by single spaces");
    else if (h.count != 3 || h.f[0] != "eg") syntax("expected 'eg <vertices> <edges>'");
    if (err.set) return fail(err);
  }
  const Fields h = split(header);
  uint32_t n = 0;
  uint64_t m = 0;
  if (!number(h.f[1], n)) {
    err.raise(line_no, "SyntaxError: line " + std::to_string(line_no) + ": malformed vertex count '" +
                           std::string(h.f[1]) + "'");
    return fail(err);
  }
  if (!number(h.f[2], m)) {
    err.raise(line_no, "SyntaxError: line " + std::to_string(line_no) + ": malformed edge count '" +
                           std::string(h.f[2]) + "'");
    return fail(err);
  }
  const uint64_t header_line = line_no;

  // chunks of the rest at line boundaries; pass 1 counts lines and records
  const unsigned T = len - pos > (1u << 22) ? host_threads() : 1u;
  std::vector<size_t> cut(T + 1, len);
  cut[0] = pos;
  for (unsigned t = 1; t < T; ++t) {
    size_t c = pos + (len - pos) * t / T;
    if (c < cut[t - 1]) c = cut[t - 1];
    const char* nl = c < len ? static_cast<const char*>(std::memchr(text + c, '\n', len - c)) : nullptr;
    cut[t] = nl ? (size_t)(nl - text) + 1 : len;
  }
  std::vector<uint64_t> lines(T, 0), recs(T, 0);
  run_threads(T, [&](unsigned t) {
    uint64_t nl = 0, nr = 0;
    for_records(text, cut[t], cut[t + 1], 0, [&](std::string_view, uint64_t ln) {
      ++nr;
      nl = ln;
      return true;
    });
    // lines: every '\n' in the chunk (+1 for an unterminated last line)
    uint64_t count = 0;
    for (size_t i = cut[t]; i < cut[t + 1]; ++i) count += text[i] == '\n';
    if (cut[t + 1] == len && len > cut[t] && text[len - 1] != '\n') ++count;
    (void)nl;
    lines[t] = count;
    recs[t] = nr;
  });
  std::vector<uint64_t> line0(T, header_line), rec0(T, 0);
  for (unsigned t = 1; t < T; ++t) {
    line0[t] = line0[t - 1] + lines[t - 1];
    rec0[t] = rec0[t - 1] + recs[t - 1];
  }
  const uint64_t total = rec0[T - 1] + recs[T - 1];
  // pass 2: parse every record into its slot
  std::vector<uint8_t> owners(n);
  std::vector<uint32_t> src(m), dst(m);
  std::vector<int64_t> w(m);
  std::vector<InputError> errs(T);
  run_threads(T, [&](unsigned t) {
    uint64_t r = rec0[t];
    InputError& e = errs[t];
    for_records(text, cut[t], cut[t + 1], line0[t], [&](std::string_view line, uint64_t ln) {
      const uint64_t i = r++;
      auto syntax = [&](const std::string& why) {
        e.raise(ln, "SyntaxError: line " + std::to_string(ln) + ": " + why);
        return false;
      };
      const Fields f = split(line);
      if (i >= (uint64_t)n + m) return syntax("unexpected record after the declared edge list");
      if (f.empty_field) return syntax("fields must be separated by single spaces");
      if (i < n) {
        if (f.count != 3 || f.f[0] != "v") return syntax("expected 'v <id> <owner>'");
        uint32_t id = 0, o = 0;
        if (!number(f.f[1], id)) return syntax("malformed vertex id '" + std::string(f.f[1]) + "'");
        if (id != i) return syntax("vertex ids must be 0..V-1 in order");
        if (!number(f.f[2], o)) return syntax("malformed owner '" + std::string(f.f[2]) + "'");
        if (o > 1) return syntax("owner must be 0 or 1");
        owners[i] = (uint8_t)o;
        return true;
      }
      const uint64_t k = i - n;
      if (f.count != 4 || f.f[0] != "e") return syntax("expected 'e <src> <dst> <weight>'");
      uint64_t s = 0, d = 0;
      int64_t wt = 0;
      if (!number(f.f[1], s)) return syntax("malformed source id '" + std::string(f.f[1]) + "'");
      if (!number(f.f[2], d)) return syntax("malformed target id '" + std::string(f.f[2]) + "'");
      if (s > UINT32_MAX) {
        e.raise(ln, "DanglingVertexIdError: edge references unknown vertex id " + std::to_string(s));
        return false;
      }
      if (d > UINT32_MAX) {
        e.raise(ln, "DanglingVertexIdError: edge references unknown vertex id " + std::to_string(d));
        return false;
      }
      if (!number(f.f[3], wt)) return syntax("malformed weight '" + std::string(f.f[3]) + "'");
      src[k] = (uint32_t)s;
      dst[k] = (uint32_t)d;
      w[k] = wt;
      return true;
    });
  });
  for (auto& e : errs)
    if (e.set) err.raise(e.line, e.msg, e.code);
  // records missing at the end of the file (the reference stops at the first
  // missing one, after any syntax error before it)
  if (!err.set && total < n)
    err.raise(~0ull, "CountMismatchError: declared " + std::to_string(n) + " vertices, found " +
                         std::to_string(total));
  else if (!err.set && total < (uint64_t)n + m)
    err.raise(~0ull, "CountMismatchError: declared " + std::to_string(m) + " edges, found " +
                         std::to_string(total - n));
  if (err.set) return fail(err);
  return build_arena(n, m, src.data(), dst.data(), w.data(), owners.data(), pinned, out);
}

inline void put_uint(std::string& out, uint64_t v) {
  char buf[24];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, (size_t)(r.ptr - buf));
}
inline void put_int(std::string& out, int64_t v) {
  char buf[24];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, (size_t)(r.ptr - buf));
}

// --------------------------------------------------------------- binary ----
// Layout (little-endian), every span 8-byte aligned:
//   0  char[8] "EGSARNA1"      8  u32 version (1)     12 u32 weight bytes (1/2/4/8)
//   16 u32 n                   20 u32 reserved        24 u64 m
//   32 i64 credit_cap          40 i64 max_abs_weight  48 u64 reserved[2]
//   64 u8 owners[n] | u64 csr_offsets[n+1] | u32 csr_targets[m] | W weights[m]
// credit_cap and max_abs_weight are recomputed on load (compute_stats) and
// must match the header.
constexpr char kMagic[8] = {'E', 'G', 'S', 'A', 'R', 'N', 'A', '1'};
constexpr uint64_t kHeader = 64;

uint64_t pad8(uint64_t x) { return (x + 7) & ~7ull; }

int weight_bytes_for(int64_t maxw) {
  return maxw <= 127 ? 1 : maxw <= 32767 ? 2 : maxw <= 2147483647LL ? 4 : 8;
}

template <class W>
void narrow(const int64_t* w, uint64_t m, std::vector<char>& buf) {
  buf.resize(m * sizeof(W));
  W* o = reinterpret_cast<W*>(buf.data());
  for (uint64_t i = 0; i < m; ++i) o[i] = (W)w[i];
}

template <class W>
void widen(const char* in, uint64_t m, int64_t* w) {
  const W* p = reinterpret_cast<const W*>(in);
  const unsigned T = m > (1u << 22) ? host_threads() : 1u;
  run_threads(T, [&](unsigned t) {
    const uint64_t lo = m * t / T, hi = m * (t + 1) / T;
    for (uint64_t i = lo; i < hi; ++i) w[i] = (int64_t)p[i];
  });
}

bool write_all(FILE* fp, const void* p, uint64_t bytes) {
  static const char zeros[8] = {0};
  if (bytes && std::fwrite(p, 1, bytes, fp) != bytes) return false;
  const uint64_t pad = pad8(bytes) - bytes;
  return pad == 0 || std::fwrite(zeros, 1, pad, fp) == pad;
}

bool read_all(FILE* fp, void* p, uint64_t bytes) {
  if (bytes && std::fread(p, 1, bytes, fp) != bytes) return false;
  const uint64_t pad = pad8(bytes) - bytes;
  return pad == 0 || std::fseek(fp, (long)pad, SEEK_CUR) == 0;
}

}  // namespace

extern "C" {

int egs_host_arena_build(uint32_t num_vertices, uint64_t num_edges, const uint32_t* src,
                         const uint32_t* dst, const int64_t* weights, const uint8_t* owners,
                         int pinned, egs_host_arena** out) {
  if (!out || (num_edges && (!src || !dst || !weights)) || (num_vertices && !owners)) {
    egs_internal_set_error("null argument");
    return EGS_ERR_INVALID_CONFIG;
  }
  try {
    return build_arena(num_vertices, num_edges, src, dst, weights, owners, pinned != 0, out);
  } catch (const std::bad_alloc&) {
    egs_internal_set_error("host allocation failed");
    return EGS_ERR_CUDA;
  }
}

int egs_arena_parse_text(const char* text, size_t len, int pinned, egs_host_arena** out) {
  if (!out || (len && !text)) {
    egs_internal_set_error("null argument");
    return EGS_ERR_INVALID_CONFIG;
  }
  try {
    return parse_text(text, len, pinned != 0, out);
  } catch (const std::bad_alloc&) {
    egs_internal_set_error("host allocation failed");
    return EGS_ERR_CUDA;
  }
}

int64_t egs_arena_write_text(const egs_arena_view* a, char* buf, size_t cap) {
  if (!a) {
    egs_internal_set_error("null arena");
    return -EGS_ERR_INVALID_CONFIG;
  }
  std::string out;
  out.reserve(16 + (size_t)a->num_vertices * 8 + (size_t)a->num_edges * 16);
  out += "eg ";
  put_uint(out, a->num_vertices);
  out += ' ';
  put_uint(out, a->num_edges);
  out += '\n';
  for (uint32_t v = 0; v < a->num_vertices; ++v) {
    out += "v ";
    put_uint(out, v);
    out += a->owners[v] == 0 ? " 0\n" : " 1\n";
  }
  for (uint32_t v = 0; v < a->num_vertices; ++v) {
    for (uint64_t i = a->csr_offsets[v]; i < a->csr_offsets[v + 1]; ++i) {
      out += "e ";
      put_uint(out, v);
      out += ' ';
      put_uint(out, a->csr_targets[i]);
      out += ' ';
      put_int(out, a->csr_weights[i]);
      out += '\n';
    }
  }
  if (buf) std::memcpy(buf, out.data(), std::min(cap, out.size()));
  return (int64_t)out.size();
}

int egs_arena_save(const egs_arena_view* a, const char* path) {
  if (!a || !path) {
    egs_internal_set_error("null argument");
    return EGS_ERR_INVALID_CONFIG;
  }
  FILE* fp = std::fopen(path, "wb");
  if (!fp) {
    egs_internal_set_error(std::string("cannot open ") + path + " for writing");
    return EGS_ERR_INPUT;
  }
  const uint32_t n = a->num_vertices;
  const uint64_t m = a->num_edges;
  const int wb = weight_bytes_for(a->max_abs_weight);
  unsigned char hdr[kHeader] = {0};
  std::memcpy(hdr, kMagic, 8);
  const uint32_t version = 1, wbu = (uint32_t)wb;
  std::memcpy(hdr + 8, &version, 4);
  std::memcpy(hdr + 12, &wbu, 4);
  std::memcpy(hdr + 16, &n, 4);
  std::memcpy(hdr + 24, &m, 8);
  std::memcpy(hdr + 32, &a->credit_cap, 8);
  std::memcpy(hdr + 40, &a->max_abs_weight, 8);
  std::vector<char> wbuf;
  if (wb == 1) narrow<int8_t>(a->csr_weights, m, wbuf);
  else if (wb == 2) narrow<int16_t>(a->csr_weights, m, wbuf);
  else if (wb == 4) narrow<int32_t>(a->csr_weights, m, wbuf);
  bool ok = write_all(fp, hdr, kHeader) && write_all(fp, a->owners, n) &&
            write_all(fp, a->csr_offsets, ((uint64_t)n + 1) * 8) &&
            write_all(fp, a->csr_targets, m * 4) &&
            (wb == 8 ? write_all(fp, a->csr_weights, m * 8) : write_all(fp, wbuf.data(), wbuf.size()));
  ok = (std::fclose(fp) == 0) && ok;
  if (!ok) {
    egs_internal_set_error(std::string("short write to ") + path);
    return EGS_ERR_INPUT;
  }
  return EGS_OK;
}

int egs_arena_load(const char* path, int pinned, egs_host_arena** out) {
  if (!path || !out) {
    egs_internal_set_error("null argument");
    return EGS_ERR_INVALID_CONFIG;
  }
  FILE* fp = std::fopen(path, "rb");
  if (!fp) {
    egs_internal_set_error(std::string("cannot open ") + path);
    return EGS_ERR_INPUT;
  }
  auto bad = [&](const std::string& why) {
    std::fclose(fp);
    egs_internal_set_error(std::string(path) + ": " + why);
    return EGS_ERR_INPUT;
  };
  unsigned char hdr[kHeader];
  if (std::fread(hdr, 1, kHeader, fp) != kHeader) return bad("truncated header");
  if (std::memcmp(hdr, kMagic, 8) != 0) return bad("not an egs binary arena (magic)");
  uint32_t version = 0, wb = 0, n = 0;
  uint64_t m = 0;
  int64_t cap = 0, maxw = 0;
  std::memcpy(&version, hdr + 8, 4);
  std::memcpy(&wb, hdr + 12, 4);
  std::memcpy(&n, hdr + 16, 4);
  std::memcpy(&m, hdr + 24, 8);
  std::memcpy(&cap, hdr + 32, 8);
  std::memcpy(&maxw, hdr + 40, 8);
  if (version != 1) return bad("unsupported version " + std::to_string(version));
  if (wb != 1 && wb != 2 && wb != 4 && wb != 8) return bad("bad weight width");
  std::fseek(fp, 0, SEEK_END);
  const uint64_t size = (uint64_t)std::ftell(fp);
  std::fseek(fp, (long)kHeader, SEEK_SET);
  const uint64_t want = kHeader + pad8(n) + pad8(((uint64_t)n + 1) * 8) + pad8(m * 4) + pad8(m * wb);
  if (size != want) return bad("size " + std::to_string(size) + " != expected " + std::to_string(want));
  egs_host_arena* a = egs_internal_arena_alloc(n, m, pinned != 0);
  if (!a) {
    std::fclose(fp);
    egs_internal_set_error("host allocation failed");
    return EGS_ERR_CUDA;
  }
  std::vector<char> wbuf;
  bool ok = read_all(fp, a->owner, n) && read_all(fp, a->off, ((uint64_t)n + 1) * 8) &&
            read_all(fp, a->dst, m * 4);
  if (ok) {
    if (wb == 8) {
      ok = read_all(fp, a->w, m * 8);
    } else {
      wbuf.resize(m * wb);
      ok = read_all(fp, wbuf.data(), m * wb);
      if (ok && wb == 1) widen<int8_t>(wbuf.data(), m, a->w);
      if (ok && wb == 2) widen<int16_t>(wbuf.data(), m, a->w);
      if (ok && wb == 4) widen<int32_t>(wbuf.data(), m, a->w);
    }
  }
  std::fclose(fp);
  std::string why;
  if (!ok) why = "short read";
  // the spans must be a GameArena: offsets from 0 to m, monotone, every row
  // non-empty, targets in range, owners 0/1
  if (why.empty() && (n == 0 ? m != 0 : (a->off[0] != 0 || a->off[n] != m))) why = "bad offsets";
  for (uint32_t v = 0; why.empty() && v < n; ++v) {
    if (a->off[v + 1] < a->off[v]) why = "offsets not monotone";
    else if (a->owner[v] > 1) why = "owner not 0/1";
  }
  if (why.empty()) {
    std::atomic<uint64_t> first_bad{~0ull};
    const unsigned T = m > (1u << 22) ? host_threads() : 1u;
    run_threads(T, [&](unsigned t) {
      const uint64_t lo = m * t / T, hi = m * (t + 1) / T;
      for (uint64_t i = lo; i < hi; ++i)
        if (a->dst[i] >= n) {
          uint64_t cur = first_bad.load();
          while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {
          }
          break;
        }
    });
    if (first_bad.load() != ~0ull)
      why = "DanglingVertexIdError: edge references unknown vertex id " +
            std::to_string(a->dst[first_bad.load()]);
  }
  if (!why.empty()) {
    egs_internal_arena_free(a);
    // a loader error keeps its "<Kind>: " prefix first
    egs_internal_set_error(why.rfind("DanglingVertexIdError: ", 0) == 0
                               ? why + " (" + path + ")"
                               : std::string(path) + ": " + why);
    return EGS_ERR_INPUT;
  }
  const int rc = egs_internal_finish_stats(a);  // totality, compute_stats
  if (rc != EGS_OK) {
    egs_internal_arena_free(a);
    return rc;
  }
  if (a->credit_cap != cap || a->max_abs_weight != maxw) {
    egs_internal_arena_free(a);
    egs_internal_set_error(std::string(path) + ": header statistics do not match the spans");
    return EGS_ERR_INPUT;
  }
  *out = a;
  return EGS_OK;
}

}  // extern "C"
