// fodg drop-in: host file formats (reference io.hpp contract): .fvecs /
// .ivecs and the CAGGRAPH container.  Little-endian hosts only.
#include <cstdio>
#include <cstring>
#include <memory>

#include "fodg/io.hpp"

namespace fodg {

namespace {

struct File {
    std::FILE* f = nullptr;
    std::string path;
    File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)), path(p) {
        if (!f)
            throw FormatError(std::string(mode[0] == 'r' ? "cannot open for reading: "
                                                         : "cannot open for writing: ") + p);
    }
    ~File() {
        if (f) std::fclose(f);
    }
    std::uint64_t size() {
        std::fseek(f, 0, SEEK_END);
        const long s = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        return s < 0 ? 0 : static_cast<std::uint64_t>(s);
    }
    void read(void* dst, std::size_t bytes) {
        if (bytes && std::fread(dst, 1, bytes, f) != bytes) throw FormatError("truncated file: " + path);
    }
    void write(const void* src, std::size_t bytes) {
        if (bytes && std::fwrite(src, 1, bytes, f) != bytes) throw FormatError("write failed: " + path);
    }
    void close_checked() {
        const int rc = std::fclose(f);
        f = nullptr;
        if (rc != 0) throw FormatError("write failed: " + path);
    }
};

constexpr char kMagic[8] = {'C', 'A', 'G', 'G', 'R', 'A', 'P', 'H'};

// records of [i32 dim][dim 4-byte values], every record the same dim
template <typename V>
std::vector<V> read_vecs(const std::string& path, std::uint32_t& dim_out) {
    File in(path, "rb");
    const std::uint64_t size = in.size();
    if (size == 0) throw FormatError("empty vecs file: " + path);
    std::int32_t dim = 0;
    in.read(&dim, 4);
    if (dim <= 0) throw FormatError("non-positive record dimension in " + path);
    const std::uint64_t rec = 4 + 4ull * static_cast<std::uint32_t>(dim);
    if (size % rec) throw FormatError("file length is not a multiple of the record size: " + path);
    const std::uint64_t n = size / rec;
    std::vector<V> out(n * static_cast<std::uint64_t>(dim));
    std::fseek(in.f, 0, SEEK_SET);
    for (std::uint64_t i = 0; i < n; ++i) {
        std::int32_t d = 0;
        in.read(&d, 4);
        if (d != dim) throw FormatError("inconsistent record dimension in " + path);
        in.read(out.data() + i * dim, 4ull * dim);
    }
    dim_out = static_cast<std::uint32_t>(dim);
    return out;
}

template <typename V>
void write_vecs(const std::string& path, const V* data, std::uint32_t rows, std::uint32_t cols) {
    File out(path, "wb");
    const std::int32_t d = static_cast<std::int32_t>(cols);
    for (std::uint32_t i = 0; i < rows; ++i) {
        out.write(&d, 4);
        out.write(data + static_cast<std::size_t>(i) * cols, 4ull * cols);
    }
    out.close_checked();
}

}  // namespace

Dataset load_fvecs(const std::string& path) {
    std::uint32_t dim = 0;
    auto data = read_vecs<float>(path, dim);
    try {
        return Dataset(dim, std::move(data));
    } catch (const UsageError& e) {
        throw FormatError(std::string(e.what()) + " (" + path + ")");
    }
}

IdMatrix load_ivecs(const std::string& path) {
    IdMatrix m;
    m.data = read_vecs<std::int32_t>(path, m.cols);
    m.rows = static_cast<std::uint32_t>(m.data.size() / m.cols);
    return m;
}

void save_fvecs(const Dataset& ds, const std::string& path) { write_vecs(path, ds.raw(), ds.size(), ds.dim()); }

void save_ivecs(const IdMatrix& m, const std::string& path) { write_vecs(path, m.data.data(), m.rows, m.cols); }

void save_graph(const Graph& g, const std::string& path) {
    for (const std::uint32_t id : g.ids) {
        if (has_parent_flag(id)) throw FormatError("save_graph: id with MSB set");
        if (id >= g.num_nodes) throw FormatError("save_graph: id out of range");
    }
    File out(path, "wb");
    const std::uint64_t n = g.num_nodes;
    const std::uint32_t d = g.degree;
    out.write(kMagic, 8);
    out.write(&n, 8);
    out.write(&d, 4);
    out.write(g.ids.data(), 4 * g.ids.size());
    out.close_checked();
}

Graph load_graph(const std::string& path) {
    File in(path, "rb");
    const std::uint64_t size = in.size();
    char magic[8];
    in.read(magic, 8);
    if (std::memcmp(magic, kMagic, 8) != 0) throw FormatError("bad graph magic in " + path);
    std::uint64_t n = 0;
    std::uint32_t d = 0;
    in.read(&n, 8);
    in.read(&d, 4);
    if (n == 0 || n > kMaxNodes || d == 0) throw FormatError("bad graph header in " + path);
    if (size != 20 + n * static_cast<std::uint64_t>(d) * 4)
        throw FormatError("graph payload size mismatch in " + path);
    Graph g;
    g.num_nodes = static_cast<std::uint32_t>(n);
    g.degree = d;
    g.ids.resize(n * static_cast<std::uint64_t>(d));
    in.read(g.ids.data(), 4 * g.ids.size());
    for (const std::uint32_t id : g.ids) {
        if (has_parent_flag(id)) throw FormatError("graph id with MSB set in " + path);
        if (id >= g.num_nodes) throw FormatError("graph id out of range in " + path);
    }
    return g;
}

}  // namespace fodg
