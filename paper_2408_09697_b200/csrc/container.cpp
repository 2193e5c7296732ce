// HGC1 graph container (container.hpp:8-19, container.cpp:47-154 of the
// reference): "HGC1" magic, u32 header length, a compact JSON header with
// sorted keys, the (src, dst) u32 pairs of every relation in dst-major CSR
// order, then the f32 row-major features of every dense type. The writer emits
// the reference's exact bytes (its JSON library dumps objects with sorted keys
// and no whitespace); the reader accepts any such file.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>

#include "host.hpp"

namespace hetgpu {

namespace {

const char kMagic[4] = {'H', 'G', 'C', '1'};

const char* storage_name(Storage s) {
  switch (s) {
    case Storage::Dense: return "dense";
    case Storage::Learnable: return "learnable";
    default: return "absent";
  }
}

Storage storage_from(const std::string& s) {
  if (s == "absent") return Storage::Absent;
  if (s == "dense") return Storage::Dense;
  if (s == "learnable") return Storage::Learnable;
  throw std::invalid_argument("unknown storage kind: " + s);
}

// ---- minimal JSON (the header's subset: objects, arrays, strings, integers, booleans)
struct Json {
  enum Kind { Null, Bool, Int, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  std::string s;
  std::vector<Json> a;
  std::map<std::string, Json> o;
  const Json& at(const std::string& k) const {
    auto it = o.find(k);
    if (kind != Obj || it == o.end()) throw std::runtime_error("container header: missing key " + k);
    return it->second;
  }
};

void dump_str(std::ostream& os, const std::string& s) {
  os << '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': os << "\\\""; break;
      case '\\': os << "\\\\"; break;
      case '\b': os << "\\b"; break;
      case '\f': os << "\\f"; break;
      case '\n': os << "\\n"; break;
      case '\r': os << "\\r"; break;
      case '\t': os << "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          os << buf;
        } else {
          os << static_cast<char>(c);
        }
    }
  }
  os << '"';
}

struct Parser {
  const std::string& t;
  std::size_t p = 0;
  explicit Parser(const std::string& text) : t(text) {}
  void ws() {
    while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p]))) ++p;
  }
  [[noreturn]] void fail() { throw std::runtime_error("container header: malformed JSON at byte " + std::to_string(p)); }
  char peek() {
    ws();
    if (p >= t.size()) fail();
    return t[p];
  }
  void expect(char c) {
    if (peek() != c) fail();
    ++p;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (p < t.size() && t[p] != '"') {
      char c = t[p++];
      if (c == '\\') {
        if (p >= t.size()) fail();
        const char e = t[p++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (p + 4 > t.size()) fail();
            const unsigned v = static_cast<unsigned>(std::stoul(t.substr(p, 4), nullptr, 16));
            p += 4;
            if (v < 0x80) {
              out += static_cast<char>(v);
            } else if (v < 0x800) {
              out += static_cast<char>(0xC0 | (v >> 6));
              out += static_cast<char>(0x80 | (v & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (v >> 12));
              out += static_cast<char>(0x80 | ((v >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (v & 0x3F));
            }
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    expect('"');
    return out;
  }
  Json value() {
    Json v;
    const char c = peek();
    if (c == '{') {
      ++p;
      v.kind = Json::Obj;
      if (peek() == '}') {
        ++p;
        return v;
      }
      while (true) {
        const std::string k = str();
        expect(':');
        v.o[k] = value();
        if (peek() == ',') {
          ++p;
          continue;
        }
        expect('}');
        return v;
      }
    }
    if (c == '[') {
      ++p;
      v.kind = Json::Arr;
      if (peek() == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.a.push_back(value());
        if (peek() == ',') {
          ++p;
          continue;
        }
        expect(']');
        return v;
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      v.s = str();
      return v;
    }
    if (t.compare(p, 4, "true") == 0) {
      p += 4;
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (t.compare(p, 5, "false") == 0) {
      p += 5;
      v.kind = Json::Bool;
      return v;
    }
    if (t.compare(p, 4, "null") == 0) {
      p += 4;
      return v;
    }
    std::size_t used = 0;
    v.kind = Json::Int;
    try {
      v.i = std::stoll(t.substr(p, 32), &used);
    } catch (...) {
      fail();
    }
    p += used;
    return v;
  }
};

template <typename T>
void put(std::ostream& os, T v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof(T));  // little-endian host
}
template <typename T>
T get(std::istream& is) {
  T v;
  is.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!is) throw std::runtime_error("container truncated");
  return v;
}

}  // namespace

std::string container_header(const Graph& g) {
  // keys in sorted order, no whitespace: the reference's header bytes
  std::ostringstream os;
  os << "{\"labels\":[";
  for (std::size_t i = 0; i < g.labels.size(); ++i) os << (i ? "," : "") << g.labels[i];
  os << "],\"node_types\":[";
  for (int t = 0; t < g.num_types(); ++t) {
    const NodeTypeInfo& nt = g.types[t];
    os << (t ? "," : "") << "{\"count\":" << nt.count << ",\"dim\":" << nt.dim << ",\"elem_bytes\":" << nt.elem_bytes
       << ",\"name\":";
    dump_str(os, nt.name);
    os << ",\"storage\":\"" << storage_name(nt.storage) << "\"}";
  }
  os << "],\"num_classes\":" << g.num_classes << ",\"relations\":[";
  for (int r = 0; r < g.num_rels(); ++r) {
    const RelationInfo& rel = g.rels[r];
    os << (r ? "," : "") << "{\"dst\":" << rel.dst_type << ",\"edges\":" << rel.adj.sources.size() << ",\"etype\":";
    dump_str(os, g.edge_type_names.at(rel.edge_type));
    os << ",\"reverse\":" << (rel.reverse ? "true" : "false") << ",\"src\":" << rel.src_type << "}";
  }
  os << "],\"target\":" << g.target << ",\"version\":1}";
  return os.str();
}

void save_container(const Graph& g, const std::string& path) {
  const std::string header = container_header(g);
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("cannot open for writing: " + path);
  os.write(kMagic, 4);
  put<std::uint32_t>(os, static_cast<std::uint32_t>(header.size()));
  os.write(header.data(), static_cast<std::streamsize>(header.size()));
  std::vector<std::uint32_t> buf;
  for (const auto& rel : g.rels) {
    const Adjacency& a = rel.adj;
    buf.clear();
    buf.reserve(2 * a.sources.size());
    for (std::size_t d = 0; d + 1 < a.offsets.size(); ++d)
      for (std::uint64_t e = a.offsets[d]; e < a.offsets[d + 1]; ++e) {
        buf.push_back(a.sources[e]);
        buf.push_back(static_cast<std::uint32_t>(d));
      }
    os.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size() * 4));
  }
  for (const auto& nt : g.types)
    if (nt.storage == Storage::Dense)
      os.write(reinterpret_cast<const char*>(nt.dense.data()), static_cast<std::streamsize>(nt.dense.size() * 4));
  if (!os) throw std::runtime_error("write failed: " + path);
}

ContainerLayout container_layout(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open: " + path);
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, kMagic, 4) != 0) throw std::runtime_error("bad container magic: " + path);
  const auto hlen = get<std::uint32_t>(is);
  std::string header(hlen, '\0');
  is.read(header.data(), hlen);
  if (!is) throw std::runtime_error("container truncated: " + path);
  Parser ps(header);
  const Json h = ps.value();
  if (h.at("version").i != 1) throw std::runtime_error("unsupported container version");
  ContainerLayout lay;
  Graph& g = lay.meta;
  for (const auto& t : h.at("node_types").a) {
    NodeTypeInfo nt;
    nt.name = t.at("name").s;
    nt.count = static_cast<std::uint64_t>(t.at("count").i);
    nt.dim = static_cast<int>(t.at("dim").i);
    nt.storage = storage_from(t.at("storage").s);
    nt.elem_bytes = static_cast<int>(t.at("elem_bytes").i);
    g.types.push_back(std::move(nt));
  }
  std::uint64_t at = 8 + static_cast<std::uint64_t>(hlen);
  for (const auto& r : h.at("relations").a) {
    RelationInfo rel;
    rel.src_type = static_cast<int>(r.at("src").i);
    rel.dst_type = static_cast<int>(r.at("dst").i);
    const std::string en = r.at("etype").s;
    auto it = std::find(g.edge_type_names.begin(), g.edge_type_names.end(), en);
    rel.edge_type = static_cast<int>(it - g.edge_type_names.begin());
    if (it == g.edge_type_names.end()) g.edge_type_names.push_back(en);
    rel.reverse = r.at("reverse").b;
    if (rel.src_type < 0 || rel.dst_type < 0 || rel.src_type >= g.num_types() || rel.dst_type >= g.num_types())
      throw std::runtime_error("container relation endpoint type out of range");
    const auto edges = static_cast<std::uint64_t>(r.at("edges").i);
    lay.rel_edges.push_back(edges);
    lay.rel_offset.push_back(at);
    at += 8 * edges;
    g.rels.push_back(std::move(rel));
  }
  for (const auto& nt : g.types) {
    lay.dense_offset.push_back(at);
    if (nt.storage == Storage::Dense) at += 4ULL * nt.count * nt.dim;
  }
  is.seekg(0, std::ios::end);
  if (static_cast<std::uint64_t>(is.tellg()) < at) throw std::runtime_error("container truncated");
  g.target = static_cast<int>(h.at("target").i);
  g.num_classes = static_cast<int>(h.at("num_classes").i);
  for (const auto& l : h.at("labels").a) g.labels.push_back(static_cast<std::int32_t>(l.i));
  return lay;
}

Graph load_container(const std::string& path) {
  ContainerLayout lay = container_layout(path);
  Graph& m = lay.meta;
  std::ifstream is(path, std::ios::binary);
  std::vector<std::string> names;
  std::vector<std::uint64_t> counts;
  for (const auto& t : m.types) {
    names.push_back(t.name);
    counts.push_back(t.count);
  }
  std::vector<int> rel_src, rel_dst;
  std::vector<std::vector<std::pair<NodeId, NodeId>>> pairs(m.rels.size());
  std::vector<std::uint32_t> buf;
  for (std::size_t r = 0; r < m.rels.size(); ++r) {
    rel_src.push_back(m.rels[r].src_type);
    rel_dst.push_back(m.rels[r].dst_type);
    buf.resize(2 * lay.rel_edges[r]);
    is.seekg(static_cast<std::streamoff>(lay.rel_offset[r]));
    is.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size() * 4));
    if (!is) throw std::runtime_error("container truncated");
    pairs[r].resize(lay.rel_edges[r]);
    for (std::size_t e = 0; e < lay.rel_edges[r]; ++e) pairs[r][e] = {buf[2 * e], buf[2 * e + 1]};
  }
  // one edge-type name per relation for assemble(); repeated names are merged below
  std::vector<std::string> rel_names;
  for (const auto& rel : m.rels) rel_names.push_back(m.edge_type_names[rel.edge_type]);
  Graph g = assemble(names, counts, rel_names, rel_src, rel_dst, pairs, m.target, m.num_classes);
  g.edge_type_names = m.edge_type_names;
  for (std::size_t r = 0; r < m.rels.size(); ++r) {
    g.rels[r].edge_type = m.rels[r].edge_type;
    g.rels[r].reverse = m.rels[r].reverse;
  }
  for (int t = 0; t < g.num_types(); ++t) {
    NodeTypeInfo& nt = g.types[t];
    nt.dim = m.types[t].dim;
    nt.storage = m.types[t].storage;
    nt.elem_bytes = m.types[t].elem_bytes;
    if (nt.storage != Storage::Dense) continue;
    nt.dense.resize(static_cast<std::size_t>(nt.count) * nt.dim);
    is.seekg(static_cast<std::streamoff>(lay.dense_offset[t]));
    is.read(reinterpret_cast<char*>(nt.dense.data()), static_cast<std::streamsize>(nt.dense.size() * 4));
    if (!is) throw std::runtime_error("container truncated");
  }
  g.labels = m.labels;
  return g;
}

}  // namespace hetgpu
