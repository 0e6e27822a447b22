// Edge-list ingest: the reference's text format and error
// behaviour (proj/src/graph.cpp:54-105 -- "src<TAB>dst" lines, '#' comments,
// LF or CRLF, first bad line reported as "line N: ...", empty input rejected,
// optional compaction of sparse ids in sorted order), read by a parallel
// byte-level parser instead of a getline loop:
//
//   1. the file is mmap'ed (a stream is slurped into one buffer);
//   2. the buffer is cut into one chunk per thread at line starts; every
//      thread scans its chunk once, counting lines and appending edges to its
//      own arrays, and stops at its first bad line;
//   3. line numbers are the per-chunk line counts prefix-summed, so the error
//      reported is the first bad line of the earliest failing chunk -- the
//      same line a sequential reader stops at;
//   4. compaction marks the ids present in a bitmap (atomic OR per 64-id
//      word) and renumbers by popcount rank, which is the sorted order of the
//      distinct ids;
//   5. the per-thread arrays go to Graph::from_edge_arrays (parallel CSR).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cstring>
#include <istream>
#include <iterator>
#include <string>
#include <thread>
#include <vector>

#include "levelrank/graph.hpp"
#include "parallel.hpp"

namespace levelrank {
inline namespace b200 {
namespace {

constexpr const char* kBadFormat = "expected \"src<TAB>dst\"";
constexpr const char* kBadRange = "vertex id out of range";

// Reads an optionally negative decimal integer at [p, e) the way
// std::from_chars(long long) accepts it: an optional '-', then at least one
// digit, consumed greedily.  Returns the end of the digits, or nullptr when
// there is no number or it does not fit in a long long.
const char* scan_int(const char* p, const char* e, long long& out) {
  const bool neg = p < e && *p == '-';
  const char* q = p + (neg ? 1 : 0);
  const char* d0 = q;
  unsigned long long v = 0;
  bool overflow = false;
  const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  for (; q < e && static_cast<unsigned>(*q - '0') < 10u; ++q) {
    const unsigned dig = static_cast<unsigned>(*q - '0');
    if (v > (lim - dig) / 10) overflow = true;
    else v = v * 10 + dig;
  }
  if (q == d0 || overflow) return nullptr;
  out = neg ? static_cast<long long>(0ull - v) : static_cast<long long>(v);
  return q;
}

struct ChunkOut {
  std::vector<VertexId> src, dst;
  long long lines = 0;      // lines seen (up to and including a bad one)
  long long bad_line = 0;   // 1-based within the chunk, 0 = none
  const char* what = nullptr;
  long long max_id = -1;
};

void scan_chunk(const char* p, const char* end, bool at_eof, ChunkOut& o) {
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<std::size_t>(end - p)));
    const char* le = nl ? nl : end;
    const char* next = nl ? nl + 1 : end;
    if (!nl && !at_eof) break;  // cannot happen: chunks end after a '\n'
    ++o.lines;
    if (le > p && le[-1] == '\r') --le;
    if (le == p || *p == '#') {
      p = next;
      continue;
    }
    long long a = 0, b = 0;
    const char* q = scan_int(p, le, a);
    if (!q || q == le || *q != '\t' || !(q = scan_int(q + 1, le, b)) || q != le) {
      o.bad_line = o.lines;
      o.what = kBadFormat;
      return;
    }
    if (a < 0 || b < 0 || a > kMaxVertexId || b > kMaxVertexId) {
      o.bad_line = o.lines;
      o.what = kBadRange;
      return;
    }
    o.src.push_back(static_cast<VertexId>(a));
    o.dst.push_back(static_cast<VertexId>(b));
    if (a > o.max_id) o.max_id = a;
    if (b > o.max_id) o.max_id = b;
    p = next;
  }
}

// Renumbers ids to their rank among the distinct ids present; returns the count.
VertexId compact_ids(std::vector<VertexId>& src, std::vector<VertexId>& dst, long long max_id) {
  const std::size_t words = static_cast<std::size_t>(max_id / 64 + 1);
  std::vector<std::uint64_t> bits(words, 0);
  const std::int64_t m = static_cast<std::int64_t>(src.size());
  detail::parallel_chunks(m, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t i = b; i < e; ++i)
      for (const VertexId v : {src[static_cast<std::size_t>(i)], dst[static_cast<std::size_t>(i)]}) {
        const std::uint64_t bit = 1ull << (v & 63);
        std::uint64_t* w = &bits[static_cast<std::size_t>(v) >> 6];
        if (!(__atomic_load_n(w, __ATOMIC_RELAXED) & bit)) __atomic_fetch_or(w, bit, __ATOMIC_RELAXED);
      }
  });
  std::vector<std::int64_t> rank(words + 1, 0);
  detail::parallel_chunks(static_cast<std::int64_t>(words), [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t k = b; k < e; ++k) rank[static_cast<std::size_t>(k)] = __builtin_popcountll(bits[static_cast<std::size_t>(k)]);
  });
  const std::int64_t distinct = detail::exclusive_scan_inplace(rank.data(), static_cast<std::int64_t>(words));
  auto id = [&](VertexId v) {
    const std::size_t w = static_cast<std::size_t>(v) >> 6;
    return static_cast<VertexId>(rank[w] + __builtin_popcountll(bits[w] & ((1ull << (v & 63)) - 1)));
  };
  detail::parallel_chunks(m, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t i = b; i < e; ++i) {
      src[static_cast<std::size_t>(i)] = id(src[static_cast<std::size_t>(i)]);
      dst[static_cast<std::size_t>(i)] = id(dst[static_cast<std::size_t>(i)]);
    }
  });
  return static_cast<VertexId>(distinct);
}

}  // namespace

Graph parse_edge_buffer(const char* data, std::size_t len, bool dense_ids, LoopPolicy policy) {
  // one chunk per thread (~4 MB minimum), each starting at a line start
  const int t = static_cast<int>(std::max<std::size_t>(
      1, std::min<std::size_t>(static_cast<std::size_t>(host_threads()), len >> 22)));
  std::vector<std::size_t> cut(static_cast<std::size_t>(t) + 1, len);
  cut[0] = 0;
  for (int i = 1; i < t; ++i) {
    std::size_t c = std::max(cut[static_cast<std::size_t>(i) - 1], len * static_cast<std::size_t>(i) / static_cast<std::size_t>(t));
    const void* nl = c < len ? std::memchr(data + c, '\n', len - c) : nullptr;
    cut[static_cast<std::size_t>(i)] = nl ? static_cast<std::size_t>(static_cast<const char*>(nl) - data) + 1 : len;
  }
  std::vector<ChunkOut> parts(static_cast<std::size_t>(t));
  {
    std::vector<std::thread> pool;
    for (int i = 0; i < t; ++i)
      pool.emplace_back([&, i] {
        const std::size_t b = cut[static_cast<std::size_t>(i)], e = cut[static_cast<std::size_t>(i) + 1];
        parts[static_cast<std::size_t>(i)].src.reserve((e - b) / 12 + 16);
        parts[static_cast<std::size_t>(i)].dst.reserve((e - b) / 12 + 16);
        scan_chunk(data + b, data + e, e == len, parts[static_cast<std::size_t>(i)]);
      });
    for (auto& th : pool) th.join();
  }
  long long lines_before = 0, max_id = -1;
  std::vector<std::int64_t> at(static_cast<std::size_t>(t) + 1, 0);
  for (int i = 0; i < t; ++i) {
    const ChunkOut& o = parts[static_cast<std::size_t>(i)];
    if (o.what) throw ParseError("line " + std::to_string(lines_before + o.bad_line) + ": " + o.what);
    lines_before += o.lines;
    max_id = std::max(max_id, o.max_id);
    at[static_cast<std::size_t>(i) + 1] = at[static_cast<std::size_t>(i)] + static_cast<std::int64_t>(o.src.size());
  }
  const std::int64_t m = at[static_cast<std::size_t>(t)];
  if (m == 0) throw ParseError("empty input: no edges");
  std::vector<VertexId> src, dst;
  if (t == 1) {
    src = std::move(parts[0].src);
    dst = std::move(parts[0].dst);
  } else {
    src.resize(static_cast<std::size_t>(m));
    dst.resize(static_cast<std::size_t>(m));
    std::vector<std::thread> pool;
    for (int i = 0; i < t; ++i)
      pool.emplace_back([&, i] {
        ChunkOut& o = parts[static_cast<std::size_t>(i)];
        std::copy(o.src.begin(), o.src.end(), src.begin() + at[static_cast<std::size_t>(i)]);
        std::copy(o.dst.begin(), o.dst.end(), dst.begin() + at[static_cast<std::size_t>(i)]);
        o.src = {};
        o.dst = {};
      });
    for (auto& th : pool) th.join();
  }
  const VertexId n = dense_ids ? static_cast<VertexId>(max_id + 1) : compact_ids(src, dst, max_id);
  return Graph::from_edge_arrays(n, src.data(), dst.data(), m, policy);
}

Graph parse_edge_list(std::istream& in, bool dense_ids, LoopPolicy policy) {
  const std::string buf{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
  return parse_edge_buffer(buf.data(), buf.size(), dense_ids, policy);
}

Graph load_edge_list(const std::string& path, bool dense_ids, LoopPolicy policy) {
  const int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) throw IoError("cannot open " + path);
  struct Closer {
    int fd;
    ~Closer() { ::close(fd); }
  } closer{fd};
  struct stat st{};
  if (::fstat(fd, &st) == 0 && S_ISREG(st.st_mode) && st.st_size > 0) {
    const std::size_t len = static_cast<std::size_t>(st.st_size);
    void* map = ::mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
    if (map != MAP_FAILED) {
      struct Unmap {
        void* p;
        std::size_t n;
        ~Unmap() { ::munmap(p, n); }
      } unmap{map, len};
      ::madvise(map, len, MADV_SEQUENTIAL | MADV_WILLNEED);
      return parse_edge_buffer(static_cast<const char*>(map), len, dense_ids, policy);
    }
  }
  // pipes, empty or unmappable files: read whatever the descriptor yields
  std::string buf;
  char tmp[1 << 16];
  for (ssize_t r; (r = ::read(fd, tmp, sizeof tmp)) > 0;) buf.append(tmp, static_cast<std::size_t>(r));
  return parse_edge_buffer(buf.data(), buf.size(), dense_ids, policy);
}

}  // namespace b200
}  // namespace levelrank
