// Graph ingest and embedding export on the host side of the path: the edge-list
// canonicalisation, the "GEMP" snapshot and the TSV writer a CLI drop-in needs.  Behaviour follows
// /root/reference/proj/src/graph.cpp:75-170 and src/io.cpp:17-46; nothing here touches the GPU.
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <string>
#include <vector>

#include "context.hpp"

using namespace gempe;

namespace {

struct parse_failure : data_error {
  parse_failure(const std::string& msg, std::uint64_t line) : data_error(msg), line(line) {}
  std::uint64_t line;
};

template <typename T>
T* to_c_array(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<std::size_t>(1, v.size()) * sizeof(T)));
  if (!p) throw data_error("out of memory");
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

void fill(gempe_graph* out, std::uint32_t n, const std::vector<std::uint32_t>& src, const std::vector<std::uint32_t>& dst,
          const std::vector<std::uint64_t>& labels) {
  out->n = n;
  out->m = src.size();
  out->src = to_c_array(src);
  out->dst = to_c_array(dst);
  out->raw_labels = labels.empty() ? nullptr : to_c_array(labels);
}

// ---- edge-list text -> canonical graph ------------------------------------------------------------------------
// Contract (SPEC of load_edge_list, /root/reference/proj/src/graph.cpp:75-133, and tests/test_graph.cpp:34-91): one
// "<id> <id>" pair of decimal u64 ids per line, any C-locale whitespace between and around them; lines whose first
// non-blank character is '#' or '%' and blank lines are skipped; a self-loop is dropped; of several lines naming the
// same undirected edge the FIRST one survives, with its orientation; ids are then renumbered 0..n-1 in order of first
// appearance in the surviving edges (source before target).  Anything else on a data line is a parse error that
// carries the 1-based line number.
//
// Built on sorting rather than on hash containers: the text is tokenised in one sweep into (low id, high id, line
// order) records, duplicates are removed by a sort on the undirected key, and the renumbering is a second sort of
// the endpoint occurrences -- O(E log E), no per-edge allocation.

inline bool blank(char ch) { return ch == ' ' || (ch >= '\t' && ch <= '\r'); }

const char* skip_blanks(const char* p, const char* stop) {
  while (p != stop && blank(*p)) ++p;
  return p;
}

const char* skip_word(const char* p, const char* stop) {
  while (p != stop && !blank(*p)) ++p;
  return p;
}

// [first, last) is a non-empty run of decimal digits that fits 64 bits
bool read_decimal(const char* first, const char* last, std::uint64_t* value) {
  if (first == last) return false;
  std::uint64_t acc = 0;
  for (; first != last; ++first) {
    const unsigned digit = static_cast<unsigned char>(*first) - static_cast<unsigned>('0');
    if (digit > 9u) return false;
    if (acc > UINT64_MAX / 10 || acc * 10 > UINT64_MAX - digit) return false;
    acc = acc * 10 + digit;
  }
  *value = acc;
  return true;
}

struct EdgeRecord {
  std::uint64_t lo, hi;  // undirected key
  std::uint32_t order;   // rank among the data lines that name an edge
  bool swapped;          // the line read "hi lo"
};

std::vector<EdgeRecord> tokenise_edge_lines(const char* text, std::uint64_t len) {
  std::vector<EdgeRecord> records;
  const char* cursor = text;
  const char* const stop = text + len;
  for (std::uint64_t line = 1; cursor != stop; ++line) {
    const void* nl = std::memchr(cursor, '\n', static_cast<std::size_t>(stop - cursor));
    const char* const eol = nl ? static_cast<const char*>(nl) : stop;
    const char* at = skip_blanks(cursor, eol);
    cursor = nl ? eol + 1 : stop;
    if (at == eol || *at == '#' || *at == '%') continue;
    std::uint64_t endpoint[2] = {0, 0};
    int seen = 0;
    for (; at != eol; at = skip_blanks(at, eol)) {
      const char* const word = at;
      at = skip_word(at, eol);
      std::uint64_t value = 0;
      if (seen == 2 || !read_decimal(word, at, &value)) {
        throw parse_failure("line " + std::to_string(line) + ": cannot read '" + std::string(word, at) +
                            "' as one of the two vertex ids of an edge", line);
      }
      endpoint[seen++] = value;
    }
    if (seen != 2) throw parse_failure("line " + std::to_string(line) + ": an edge needs two vertex ids", line);
    if (endpoint[0] == endpoint[1]) continue;
    if (records.size() >= 0xffffffffull) throw data_error("edge list exceeds 2^32 lines");
    const bool swapped = endpoint[0] > endpoint[1];
    records.push_back({swapped ? endpoint[1] : endpoint[0], swapped ? endpoint[0] : endpoint[1],
                       static_cast<std::uint32_t>(records.size()), swapped});
  }
  return records;
}

void parse_edge_list(const char* text, std::uint64_t len, gempe_graph* out) {
  std::vector<EdgeRecord> records = tokenise_edge_lines(text, len);
  // duplicates: group by undirected key, the earliest line of every group stays; then back to line order
  std::sort(records.begin(), records.end(), [](const EdgeRecord& x, const EdgeRecord& y) {
    return x.lo != y.lo ? x.lo < y.lo : (x.hi != y.hi ? x.hi < y.hi : x.order < y.order);
  });
  records.erase(std::unique(records.begin(), records.end(),
                            [](const EdgeRecord& x, const EdgeRecord& y) { return x.lo == y.lo && x.hi == y.hi; }),
                records.end());
  std::sort(records.begin(), records.end(), [](const EdgeRecord& x, const EdgeRecord& y) { return x.order < y.order; });
  if (records.empty()) throw data_error("the edge list holds no edge (only comments, blanks, self-loops)");

  // renumbering: occurrence 2e is the source of surviving edge e, 2e+1 its target; a raw id gets the rank of its first
  // occurrence among the first occurrences of all ids
  const std::size_t edges = records.size();
  struct Occurrence { std::uint64_t raw; std::uint64_t where; };
  std::vector<Occurrence> occ(2 * edges);
  for (std::size_t e = 0; e < edges; ++e) {
    const EdgeRecord& r = records[e];
    occ[2 * e] = {r.swapped ? r.hi : r.lo, 2 * e};
    occ[2 * e + 1] = {r.swapped ? r.lo : r.hi, 2 * e + 1};
  }
  std::sort(occ.begin(), occ.end(), [](const Occurrence& x, const Occurrence& y) {
    return x.raw != y.raw ? x.raw < y.raw : x.where < y.where;
  });
  std::vector<Occurrence> firsts;  // one per distinct raw id: (raw, first occurrence)
  for (const Occurrence& o : occ) {
    if (firsts.empty() || firsts.back().raw != o.raw) firsts.push_back(o);
  }
  if (firsts.size() > 0xffffffffull) throw data_error("more than 2^32 distinct vertex ids");
  std::vector<std::uint32_t> by_appearance(firsts.size());
  std::iota(by_appearance.begin(), by_appearance.end(), 0u);
  std::sort(by_appearance.begin(), by_appearance.end(),
            [&](std::uint32_t x, std::uint32_t y) { return firsts[x].where < firsts[y].where; });
  std::vector<std::uint32_t> new_id(firsts.size());
  std::vector<std::uint64_t> labels(firsts.size());
  for (std::uint32_t rank = 0; rank < by_appearance.size(); ++rank) {
    new_id[by_appearance[rank]] = rank;
    labels[rank] = firsts[by_appearance[rank]].raw;
  }
  auto lookup = [&](std::uint64_t raw) {
    const auto it = std::lower_bound(firsts.begin(), firsts.end(), raw,
                                     [](const Occurrence& o, std::uint64_t v) { return o.raw < v; });
    return new_id[static_cast<std::size_t>(it - firsts.begin())];
  };
  std::vector<std::uint32_t> src(edges), dst(edges);
  for (std::size_t e = 0; e < edges; ++e) {
    const EdgeRecord& r = records[e];
    src[e] = lookup(r.swapped ? r.hi : r.lo);
    dst[e] = lookup(r.swapped ? r.lo : r.hi);
  }
  fill(out, static_cast<std::uint32_t>(firsts.size()), src, dst, labels);
}

std::uint64_t le(const unsigned char* p, int bytes) {
  std::uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(p[i]) << (8 * i);
  return v;
}

// load_graph_snapshot (graph.cpp:149-170): "GEMP", u32 n, u64 m, src[m], dst[m], little-endian
void parse_snapshot(const unsigned char* b, std::uint64_t len, gempe_graph* out) {
  if (len < 4 || std::memcmp(b, "GEMP", 4) != 0) throw data_error("bad snapshot magic");
  if (len < 16) throw data_error("truncated snapshot");
  const std::uint32_t n = static_cast<std::uint32_t>(le(b + 4, 4));
  const std::uint64_t m = le(b + 8, 8);
  if (m == 0) throw data_error("snapshot holds no edges");
  const std::uint64_t pairs = static_cast<std::uint64_t>(n) * (n > 0 ? n - 1 : 0) / 2;
  if (m > pairs) throw data_error("snapshot edge count exceeds pair count");
  if ((len - 16) / 8 < m) throw data_error("truncated snapshot");
  std::vector<std::uint32_t> src(m), dst(m);
  for (std::uint64_t e = 0; e < m; ++e) src[e] = static_cast<std::uint32_t>(le(b + 16 + 4 * e, 4));
  for (std::uint64_t e = 0; e < m; ++e) dst[e] = static_cast<std::uint32_t>(le(b + 16 + 4 * (m + e), 4));
  for (std::uint64_t e = 0; e < m; ++e) {
    if (src[e] >= n || dst[e] >= n || src[e] == dst[e]) throw data_error("snapshot edge out of range");
  }
  fill(out, n, src, dst, {});
}

template <typename Fn>
int guarded_io(std::uint64_t* error_line, Fn&& fn) {
  if (error_line) *error_line = 0;
  try {
    fn();
    return GEMPE_OK;
  } catch (const parse_failure& e) {
    if (error_line) *error_line = e.line;
    set_create_error(e.what());
    return GEMPE_ERR_DATA;
  } catch (const config_error& e) {
    set_create_error(e.what());
    return GEMPE_ERR_CONFIG;
  } catch (const std::exception& e) {
    set_create_error(e.what());
    return GEMPE_ERR_DATA;
  }
}

}  // namespace

extern "C" {

int gempe_parse_edge_list(const char* text, std::uint64_t len, gempe_graph* out, std::uint64_t* error_line) {
  return guarded_io(error_line, [&] {
    if (!out) throw config_error("null graph");
    std::memset(out, 0, sizeof *out);
    parse_edge_list(text, len, out);
  });
}

int gempe_parse_graph_snapshot(const void* bytes, std::uint64_t len, gempe_graph* out) {
  return guarded_io(nullptr, [&] {
    if (!out) throw config_error("null graph");
    std::memset(out, 0, sizeof *out);
    parse_snapshot(static_cast<const unsigned char*>(bytes), len, out);
  });
}

// looks_like_snapshot ? load_graph_snapshot : load_edge_list  (tools/embed_main.cpp:150-153)
int gempe_load_graph_file(const char* path, gempe_graph* out, std::uint64_t* error_line) {
  return guarded_io(error_line, [&] {
    if (!out || !path) throw config_error("null argument");
    std::memset(out, 0, sizeof *out);
    std::ifstream in(path, std::ios::binary);
    if (!in) throw data_error(std::string("cannot open ") + path);
    std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (bytes.size() >= 4 && std::memcmp(bytes.data(), "GEMP", 4) == 0) {
      parse_snapshot(reinterpret_cast<const unsigned char*>(bytes.data()), bytes.size(), out);
    } else {
      parse_edge_list(bytes.data(), bytes.size(), out);
    }
  });
}

int gempe_write_graph_snapshot(const char* path, std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                               const std::uint32_t* dst) {
  return guarded_io(nullptr, [&] {  // save_graph_snapshot (graph.cpp:141-147)
    std::ofstream o(path, std::ios::binary);
    if (!o) throw data_error(std::string("cannot open ") + path);
    auto put = [&](std::uint64_t v, int bytes) {
      char b[8];
      for (int i = 0; i < bytes; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
      o.write(b, bytes);
    };
    o.write("GEMP", 4);
    put(n, 4);
    put(m, 8);
    for (std::uint64_t e = 0; e < m; ++e) put(src[e], 4);
    for (std::uint64_t e = 0; e < m; ++e) put(dst[e], 4);
    if (!o) throw data_error("short write");
  });
}

void gempe_graph_free(gempe_graph* g) {
  if (!g) return;
  std::free(g->src);
  std::free(g->dst);
  std::free(g->raw_labels);
  std::memset(g, 0, sizeof *g);
}

// write_embedding_tsv (io.cpp:17-46): "#id<TAB>x0..." header, rows in ascending label order, "%.6g" coordinates;
// with perm_forward the row of vertex v is coords[perm_forward[v]].
int gempe_write_embedding_tsv(const char* path, std::uint32_t n, std::uint32_t dim, const float* coords,
                              const std::uint64_t* labels, const std::uint32_t* perm_forward) {
  return guarded_io(nullptr, [&] {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw data_error(std::string("cannot open ") + path);
    std::fputs("#id", f);
    for (std::uint32_t k = 0; k < dim; ++k) std::fprintf(f, "\tx%u", k);
    std::fputc('\n', f);
    std::vector<std::uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    if (labels) std::sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) { return labels[a] < labels[b]; });
    for (std::uint32_t v : order) {
      const std::uint32_t row = perm_forward ? perm_forward[v] : v;
      std::fprintf(f, "%" PRIu64, labels ? labels[v] : static_cast<std::uint64_t>(v));
      for (std::uint32_t k = 0; k < dim; ++k) {
        std::fprintf(f, "\t%.6g", static_cast<double>(coords[static_cast<std::size_t>(row) * dim + k]));
      }
      std::fputc('\n', f);
    }
    if (std::fclose(f) != 0) throw data_error("short write");
  });
}

}  // extern "C"
