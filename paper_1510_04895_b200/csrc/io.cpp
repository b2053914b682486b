// On-disk formats around the hot path:
//  * Matrix Market coordinate read/write (matrix_market.cpp:19-115): real,
//    integer, complex fields; general / symmetric / hermitian storage, the
//    latter expanded to full storage; duplicates summed in file order as the
//    reference's Builder does (sparse_matrix.hpp:61-79).  Writes 17 digits so a
//    write -> read round trip is exact.
//  * .cbfd block dumps (block_vector.hpp:63-96): u32 magic "CBFD", u64 dim,
//    u32 width, u32 kind, raw row-major payload.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "capi_common.hpp"

namespace cfd {

namespace {

// whitespace tokens of one line; a token must parse completely
struct Tokens {
    std::vector<std::string> t;
    explicit Tokens(const std::string& line) {
        size_t p = 0;
        while (p < line.size()) {
            while (p < line.size() && std::isspace(static_cast<unsigned char>(line[p]))) ++p;
            size_t q = p;
            while (q < line.size() && !std::isspace(static_cast<unsigned char>(line[q]))) ++q;
            if (q > p) t.emplace_back(line.substr(p, q - p));
            p = q;
        }
    }
    bool integer(size_t k, int64_t& v) const {
        if (k >= t.size()) return false;
        char* e = nullptr;
        v = std::strtoll(t[k].c_str(), &e, 10);
        return *e == '\0';
    }
    bool real(size_t k, double& v) const {  // strtod: the conversion istream >> double uses
        if (k >= t.size()) return false;
        char* e = nullptr;
        v = std::strtod(t[k].c_str(), &e);
        return e != t[k].c_str();
    }
};

struct Trip {
    int64_t i, j;
    double re, im;
};

// triplets -> CSR with ascending columns, duplicates summed in insertion order from S{}
HostCsr build_csr(std::vector<Trip>& t, int64_t dim, int kind) {
    std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
        return a.i != b.i ? a.i < b.i : a.j < b.j;
    });
    HostCsr h;
    h.kind = kind;
    h.dim = dim;
    h.rows = dim;
    h.offs.assign(static_cast<size_t>(dim) + 1, 0);
    for (size_t k = 0; k < t.size();) {
        size_t e = k;
        double re = 0.0, im = 0.0;
        for (; e < t.size() && t[e].i == t[k].i && t[e].j == t[k].j; ++e) {
            re += t[e].re;
            im += t[e].im;
        }
        h.cols.push_back(t[k].j);
        h.vals.push_back(re);
        if (kind) h.vals.push_back(im);
        h.offs[t[k].i + 1] += 1;
        k = e;
    }
    for (int64_t r = 0; r < dim; ++r) h.offs[r + 1] += h.offs[r];
    return h;
}

enum class Storage { General, Symmetric, Hermitian };

}  // namespace

HostCsr read_matrix_market(const std::string& path, bool* hermitian) {
    std::ifstream in(path);
    if (!in) fail(CHEBFD_ERR_RUNTIME, "cannot open " + path);
    std::string line;
    if (!std::getline(in, line) || line.compare(0, 14, "%%MatrixMarket") != 0)
        fail(CHEBFD_ERR_RUNTIME, path + ": missing MatrixMarket banner");
    for (char& ch : line) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    const Tokens banner(line);  // %%matrixmarket object format field symmetry
    auto word = [&](size_t k) { return k < banner.t.size() ? banner.t[k] : std::string(); };
    if (word(1) != "matrix" || word(2) != "coordinate")
        fail(CHEBFD_ERR_RUNTIME, path + ": only coordinate matrices are supported");
    const std::string sym = word(4);
    Storage storage;
    if (sym == "general")
        storage = Storage::General;
    else if (sym == "symmetric")
        storage = Storage::Symmetric;
    else if (sym == "hermitian")
        storage = Storage::Hermitian;
    else
        fail(CHEBFD_ERR_RUNTIME, path + ": unsupported symmetry '" + sym + "'");
    const std::string field = word(3);
    int kind;
    if (field == "real" || field == "integer")
        kind = CHEBFD_REAL64;
    else if (field == "complex")
        kind = CHEBFD_COMPLEX128;
    else
        fail(CHEBFD_ERR_RUNTIME, path + ": unsupported field '" + field + "'");

    auto next_data_line = [&]() -> bool {
        while (std::getline(in, line))
            if (!line.empty() && line[0] != '%') return true;
        return false;
    };
    int64_t n = 0, m = 0, declared = 0;
    if (next_data_line()) {
        const Tokens sz(line);
        if (!sz.integer(0, n) || !sz.integer(1, m) || !sz.integer(2, declared))
            fail(CHEBFD_ERR_RUNTIME, path + ": malformed size line");
    }
    if (n != m) fail(CHEBFD_ERR_RUNTIME, path + ": matrix is not square");
    if (n < 0) fail(CHEBFD_ERR_RUNTIME, path + ": negative dimension");

    std::vector<Trip> trips;
    trips.reserve(static_cast<size_t>(std::max<int64_t>(declared, 0)) *
                  (storage == Storage::General ? 1 : 2));
    int64_t got = 0;
    for (; got < declared && next_data_line(); ++got) {
        const Tokens e(line);
        int64_t i, j;
        double re = 0.0, im = 0.0;
        if (!e.integer(0, i) || !e.integer(1, j))
            fail(CHEBFD_ERR_RUNTIME, path + ": malformed entry line");
        if (!e.real(2, re)) fail(CHEBFD_ERR_RUNTIME, path + ": missing value");
        if (kind && !e.real(3, im)) fail(CHEBFD_ERR_RUNTIME, path + ": missing imaginary part");
        i -= 1;  // 1-based on disk
        j -= 1;
        if (i < 0 || i >= n || j < 0 || j >= n)  // Builder::add (sparse_matrix.hpp:61-63)
            fail(CHEBFD_ERR_OUT_OF_RANGE, "SparseMatrix::Builder: index out of range");
        trips.push_back({i, j, re, im});
        if (i == j || storage == Storage::General) continue;
        trips.push_back({j, i, re, storage == Storage::Hermitian ? -im : im});
    }
    if (got != declared) fail(CHEBFD_ERR_RUNTIME, path + ": fewer entries than declared");
    if (hermitian) *hermitian = storage != Storage::General;
    return build_csr(trips, n, kind);
}

void write_matrix_market(const std::string& path, int kind, int64_t dim, const int64_t* offs,
                         const int64_t* cols, const double* vals, bool herm) {
    // symmetric / Hermitian storage keeps the lower triangle (j <= i)
    auto stored = [&](int64_t i, int64_t p) { return !herm || cols[p] <= i; };
    int64_t kept = 0;
    for (int64_t i = 0; i < dim; ++i)
        for (int64_t p = offs[i]; p < offs[i + 1]; ++p) kept += stored(i, p);
    std::string body;
    body.reserve(static_cast<size_t>(kept) * (kind ? 56 : 34) + 128);
    char buf[128];
    std::snprintf(buf, sizeof buf, "%%%%MatrixMarket matrix coordinate %s %s\n%lld %lld %lld\n",
                  kind ? "complex" : "real",
                  herm ? (kind ? "hermitian" : "symmetric") : "general",
                  static_cast<long long>(dim), static_cast<long long>(dim),
                  static_cast<long long>(kept));
    body += buf;
    for (int64_t i = 0; i < dim; ++i)
        for (int64_t p = offs[i]; p < offs[i + 1]; ++p) {
            if (!stored(i, p)) continue;
            // %.17g == ostream precision(17) default float format: exact round trip
            int n = kind ? std::snprintf(buf, sizeof buf, "%lld %lld %.17g %.17g\n",
                                         static_cast<long long>(i + 1),
                                         static_cast<long long>(cols[p] + 1), vals[2 * p],
                                         vals[2 * p + 1])
                         : std::snprintf(buf, sizeof buf, "%lld %lld %.17g\n",
                                         static_cast<long long>(i + 1),
                                         static_cast<long long>(cols[p] + 1), vals[p]);
            body.append(buf, static_cast<size_t>(n));
        }
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) fail(CHEBFD_ERR_RUNTIME, "cannot open " + path + " for writing");
    const bool ok = std::fwrite(body.data(), 1, body.size(), f) == body.size();
    if (std::fclose(f) != 0 || !ok) fail(CHEBFD_ERR_RUNTIME, "write failed: " + path);
}

constexpr uint32_t kCbfdMagic = 0x44464243u;  // "CBFD"

void save_cbfd(const std::string& path, int kind, uint64_t dim, uint32_t width, const void* data) {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(CHEBFD_ERR_RUNTIME, "BlockVector::save: cannot open " + path);
    const uint32_t magic = kCbfdMagic, k = static_cast<uint32_t>(kind);
    out.write(reinterpret_cast<const char*>(&magic), 4);
    out.write(reinterpret_cast<const char*>(&dim), 8);
    out.write(reinterpret_cast<const char*>(&width), 4);
    out.write(reinterpret_cast<const char*>(&k), 4);
    out.write(static_cast<const char*>(data),
              static_cast<std::streamsize>(dim * width * (kind ? 16 : 8)));
    if (!out) fail(CHEBFD_ERR_RUNTIME, "BlockVector::save: write failed");
}

// header only (data == nullptr) or header + payload into data
void load_cbfd(const std::string& path, int* kind, uint64_t* dim, uint32_t* width, void* data) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(CHEBFD_ERR_RUNTIME, "BlockVector::load: cannot open " + path);
    uint32_t magic = 0, k = 0, w = 0;
    uint64_t d = 0;
    in.read(reinterpret_cast<char*>(&magic), 4);
    in.read(reinterpret_cast<char*>(&d), 8);
    in.read(reinterpret_cast<char*>(&w), 4);
    in.read(reinterpret_cast<char*>(&k), 4);
    if (!in || magic != kCbfdMagic) fail(CHEBFD_ERR_RUNTIME, "BlockVector::load: bad header");
    if (k > 1) fail(CHEBFD_ERR_RUNTIME, "BlockVector::load: scalar kind mismatch");
    *kind = static_cast<int>(k);
    *dim = d;
    *width = w;
    if (!data) return;
    in.read(static_cast<char*>(data), static_cast<std::streamsize>(d * w * (k ? 16 : 8)));
    if (!in) fail(CHEBFD_ERR_RUNTIME, "BlockVector::load: truncated payload");
}

}  // namespace cfd

using namespace cfd;

extern "C" {

int chebfd_read_matrix_market(const char* path, int* kind, int64_t* dim, int64_t* nnz,
                              int64_t* offs, int64_t* cols, void* vals, int* hermitian) {
    return guard([&] {
        bool herm = true;
        HostCsr h = read_matrix_market(path, &herm);
        *kind = h.kind;
        *dim = h.dim;
        *nnz = static_cast<int64_t>(h.cols.size());
        if (hermitian) *hermitian = herm ? 1 : 0;
        if (offs) {
            std::memcpy(offs, h.offs.data(), sizeof(int64_t) * h.offs.size());
            std::memcpy(cols, h.cols.data(), sizeof(int64_t) * h.cols.size());
            std::memcpy(vals, h.vals.data(), sizeof(double) * h.vals.size());
        }
    });
}

int chebfd_write_matrix_market(const char* path, int kind, int64_t dim, const int64_t* offs,
                               const int64_t* cols, const void* vals, int hermitian) {
    return guard([&] {
        require(kind == CHEBFD_REAL64 || kind == CHEBFD_COMPLEX128, "bad scalar kind");
        write_matrix_market(path, kind, dim, offs, cols, static_cast<const double*>(vals),
                            hermitian != 0);
    });
}

int chebfd_cbfd_save(const char* path, int kind, uint64_t dim, uint32_t width, const void* data) {
    return guard([&] { save_cbfd(path, kind, dim, width, data); });
}

int chebfd_cbfd_load(const char* path, int* kind, uint64_t* dim, uint32_t* width, void* data) {
    return guard([&] { load_cbfd(path, kind, dim, width, data); });
}

}  // extern "C"

// ---- device objects <-> files (single-GPU contexts: the files hold the whole D x nb block) ----
extern "C" {

int chebfd_matrix_from_matrix_market(chebfd_ctx* ctx, const char* path, chebfd_matrix** out) {
    HostCsr h;
    const int st = guard([&] { h = read_matrix_market(path, nullptr); });
    if (st != CHEBFD_OK) return st;
    return chebfd_matrix_from_csr(ctx, h.kind, h.dim, h.offs.data(), h.cols.data(),
                                  h.vals.data(), out);
}

int chebfd_block_save(const chebfd_block* b, const char* path) {
    return guard([&] {
        const Block* x = reinterpret_cast<const Block*>(b);
        if (x->rows != x->dim_global)
            fail(CHEBFD_ERR_UNSUPPORTED, "BlockVector::save: block is distributed over ranks");
        std::vector<double> host(static_cast<size_t>(x->rows * x->width) * (x->kind ? 2 : 1));
        const int st = chebfd_block_download(b, host.data());
        if (st != CHEBFD_OK) throw Error(st, g_last_error);
        save_cbfd(path, x->kind, static_cast<uint64_t>(x->rows), static_cast<uint32_t>(x->width),
                  host.data());
    });
}

int chebfd_block_load(chebfd_matrix* a, const char* path, chebfd_block** out) {
    return guard([&] {
        const Matrix* m = reinterpret_cast<const Matrix*>(a);
        int kind = 0;
        uint64_t dim = 0;
        uint32_t width = 0;
        load_cbfd(path, &kind, &dim, &width, nullptr);
        if (kind != m->kind) fail(CHEBFD_ERR_RUNTIME, "BlockVector::load: scalar kind mismatch");
        if (static_cast<int64_t>(dim) != m->part.dim)
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "BlockVector::load: dimension does not match matrix");
        if (m->part.local != m->part.dim)
            fail(CHEBFD_ERR_UNSUPPORTED, "BlockVector::load: matrix is distributed over ranks");
        std::vector<double> host(static_cast<size_t>(dim) * width * (kind ? 2 : 1));
        load_cbfd(path, &kind, &dim, &width, host.data());
        chebfd_block* blk = nullptr;
        int st = chebfd_block_create(a, width, &blk);
        if (st == CHEBFD_OK) st = chebfd_block_upload(blk, host.data());
        if (st != CHEBFD_OK) {
            const std::string msg = g_last_error;
            if (blk) chebfd_block_destroy(blk);
            throw Error(st, msg);
        }
        *out = blk;
    });
}

}  // extern "C"
