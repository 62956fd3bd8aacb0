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
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "context.hpp"

using namespace gempe;

namespace {

struct parse_failure : data_error {
  parse_failure(const std::string& msg, std::uint64_t line) : data_error(msg), line(line) {}
  std::uint64_t line;
};

bool is_space(unsigned char ch) { return ch == ' ' || (ch >= '\t' && ch <= '\r'); }  // std::isspace, "C" locale

struct PairKeyHash {
  std::size_t operator()(const std::pair<std::uint64_t, std::uint64_t>& p) const {
    return static_cast<std::size_t>(splitmix64(p.first * 0x100000001b3ull ^ p.second));
  }
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

// load_edge_list (graph.cpp:75-133): "i<ws>j" lines, '#'/'%' comments and blank lines skipped, self-loops dropped,
// duplicate undirected edges merged (first occurrence and its orientation kept), ids compacted in first-appearance order.
void parse_edge_list(const char* text, std::uint64_t len, gempe_graph* out) {
  std::vector<std::pair<std::uint64_t, std::uint64_t>> raw_edges;
  std::unordered_set<std::pair<std::uint64_t, std::uint64_t>, PairKeyHash> seen;
  std::uint64_t line_no = 0, at = 0;
  while (at < len) {
    std::uint64_t end = at;
    while (end < len && text[end] != '\n') ++end;
    ++line_no;
    std::uint64_t pos = at;
    const std::uint64_t stop = end;
    at = end + 1;  // a final line without '\n' is still a line; an empty tail after the last '\n' is not
    while (pos < stop && is_space(static_cast<unsigned char>(text[pos]))) ++pos;
    if (pos == stop) continue;
    if (text[pos] == '#' || text[pos] == '%') continue;
    std::uint64_t ids[2] = {0, 0};
    int count = 0;
    while (pos < stop) {
      while (pos < stop && is_space(static_cast<unsigned char>(text[pos]))) ++pos;
      if (pos == stop) break;
      const std::uint64_t start = pos;
      while (pos < stop && !is_space(static_cast<unsigned char>(text[pos]))) ++pos;
      std::uint64_t v = 0;
      bool ok = count < 2 && pos > start;
      for (std::uint64_t q = start; ok && q < pos; ++q) {
        const char ch = text[q];
        if (ch < '0' || ch > '9') ok = false;
        else {
          const std::uint64_t digit = static_cast<std::uint64_t>(ch - '0');
          if (v > (UINT64_MAX - digit) / 10) ok = false;
          else v = v * 10 + digit;
        }
      }
      if (!ok) {
        throw parse_failure("malformed edge line " + std::to_string(line_no) + ": '" + std::string(text + start, pos - start) + "'",
                            line_no);
      }
      ids[count++] = v;
    }
    if (count != 2) throw parse_failure("expected two vertex ids on line " + std::to_string(line_no), line_no);
    if (ids[0] == ids[1]) continue;
    if (!seen.insert({std::min(ids[0], ids[1]), std::max(ids[0], ids[1])}).second) continue;
    raw_edges.emplace_back(ids[0], ids[1]);
  }
  if (raw_edges.empty()) throw data_error("no edges after canonicalization");
  std::unordered_map<std::uint64_t, std::uint32_t> compact;
  compact.reserve(raw_edges.size() * 2);
  std::vector<std::uint64_t> labels;
  std::vector<std::uint32_t> src, dst;
  src.reserve(raw_edges.size());
  dst.reserve(raw_edges.size());
  auto id_of = [&](std::uint64_t raw) {
    auto [it, inserted] = compact.try_emplace(raw, static_cast<std::uint32_t>(compact.size()));
    if (inserted) labels.push_back(raw);
    return it->second;
  };
  for (const auto& [a, b] : raw_edges) {
    const std::uint32_t ia = id_of(a), ib = id_of(b);
    src.push_back(ia);
    dst.push_back(ib);
  }
  fill(out, static_cast<std::uint32_t>(compact.size()), src, dst, labels);
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
