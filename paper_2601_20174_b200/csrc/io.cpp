// paper_2601_20174_b200/csrc/io.cpp — the reference's on-disk inputs for the
// solver path (include/nlsp_io.h): MatrixMarket matrices and
// `nlsp gen` instance directories, read into the reference's CSR layout for
// nlsp_csr_upload.
//
// The reference reads with iostreams (sparse.hpp:168-194, csv.hpp,
// instance_io.hpp:137-185). Here the file is read in one block and scanned
// with a cursor that reproduces `istream >> size_t` / `istream >> double`
// token by token (libstdc++ num_get: the same accepted characters, the same
// strtod conversion and failure rules), so every file the reference accepts
// loads to the same bits and every file it rejects fails with the same error
// class. The triplet -> CSR step is a counting sort by row plus an insertion
// sort by column inside each row (stable), O(nnz) for the sorted files the
// reference writes, instead of a comparison sort of all triplets.
#include "nlsp_io.h"

#include "host_rng.hpp"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_err;

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return NLSP_IO_OK;
    } catch (const IoError& e) {
        g_err = e.what();
        return NLSP_IO_E_IO;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return NLSP_IO_E_VALIDATION;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return NLSP_IO_E_IO;
    } catch (const std::exception& e) {  // std::stod / stoull failures in the reference
        g_err = e.what();
        return NLSP_IO_E_VALIDATION;
    }
}

bool read_file(const std::string& path, std::string& buf) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    buf.clear();
    char tmp[1 << 16];
    size_t got;
    while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.append(tmp, got);
    std::fclose(f);
    return true;
}

// std::getline over an in-memory buffer
struct Lines {
    const std::string& s;
    size_t pos = 0;
    bool next(std::string& line) {
        if (pos >= s.size()) return false;
        const size_t e = s.find('\n', pos);
        if (e == std::string::npos) {
            line.assign(s, pos, std::string::npos);
            pos = s.size();
        } else {
            line.assign(s, pos, e - pos);
            pos = e + 1;
        }
        return true;
    }
};

inline bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// istream-style extraction from [p, end): skips leading whitespace; on
// failure the stream is "failed" and every later extraction fails too.
struct Cursor {
    const char* p;
    const char* end;
    bool fail = false;

    void skip_ws() {
        while (p < end && is_space(*p)) ++p;
    }
    // operator>>(size_t&): optional sign, decimal digits; '-' negates modulo
    // 2^64 (strtoull semantics); overflow fails
    unsigned long long u64() {
        if (fail) return 0;
        skip_ws();
        bool neg = false;
        if (p < end && (*p == '+' || *p == '-')) {
            neg = *p == '-';
            ++p;
        }
        unsigned long long v = 0;
        bool digits = false, overflow = false;
        while (p < end && *p >= '0' && *p <= '9') {
            const unsigned d = (unsigned)(*p - '0');
            if (v > (std::numeric_limits<unsigned long long>::max() - d) / 10) overflow = true;
            v = v * 10 + d;
            digits = true;
            ++p;
        }
        if (!digits || overflow) {
            fail = true;
            return overflow ? std::numeric_limits<unsigned long long>::max() : 0;
        }
        return neg ? (unsigned long long)(0 - v) : v;
    }
    // operator>>(double&): [sign] digits [. digits] [(e|E) [sign] digits],
    // 'e' accepted only after mantissa digits; converted by strtod, which must
    // consume the whole accumulated text; +-inf results fail
    double f64() {
        if (fail) return 0.0;
        skip_ws();
        char buf[512];
        size_t n = 0;
        auto put = [&](char c) {
            if (n + 1 < sizeof(buf)) buf[n++] = c;
        };
        if (p < end && (*p == '+' || *p == '-')) put(*p++);
        bool mant = false, dot = false;
        while (p < end) {
            const char c = *p;
            if (c >= '0' && c <= '9') {
                mant = true;
                put(c);
                ++p;
            } else if (c == '.' && !dot) {
                dot = true;
                put(c);
                ++p;
            } else {
                break;
            }
        }
        if (mant && p < end && (*p == 'e' || *p == 'E')) {
            put(*p++);
            if (p < end && (*p == '+' || *p == '-')) put(*p++);
            while (p < end && *p >= '0' && *p <= '9') put(*p++);
        }
        buf[n] = '\0';
        char* q = nullptr;
        const double v = std::strtod(buf, &q);
        if (n == 0 || q == buf || *q != '\0' || std::isinf(v)) {
            fail = true;
            return 0.0;
        }
        return v;
    }
};

struct Trip {
    unsigned long long i, j;
    double v;
};

// SparseCsrMatrix::from_triplets (sparse.hpp:24-53)
void from_triplets(unsigned long long dim, const std::vector<Trip>& t, nlsp_host_csr* out) {
    // a size line such as "-1 -1 0" parses to 2^64 - 1 (istream >> size_t
    // wraps negatives): dim + 1 would wrap to an empty row_ptr. Dimensions past
    // the device limit (nlsp_csr_upload: n < 2^31) are rejected before anything
    // is allocated.
    if (dim >= (1ull << 31)) throw ValidationError("matrix dimension exceeds 2^31 - 1");
    for (const Trip& e : t)
        if (e.i >= dim || e.j >= dim) throw ValidationError("triplet index out of range");
    std::vector<unsigned long long> start(dim + 1, 0);
    for (const Trip& e : t) ++start[e.i + 1];
    for (unsigned long long r = 0; r < dim; ++r) start[r + 1] += start[r];
    std::vector<unsigned long long> cols(t.size());
    std::vector<double> vals(t.size());
    {
        std::vector<unsigned long long> fill(start.begin(), start.end() - 1);
        for (const Trip& e : t) {
            const unsigned long long at = fill[e.i]++;
            cols[at] = e.j;
            vals[at] = e.v;
        }
    }
    std::vector<unsigned long long> rp(dim + 1, 0), ci;
    std::vector<double> v;
    ci.reserve(t.size());
    v.reserve(t.size());
    for (unsigned long long r = 0; r < dim; ++r) {
        const unsigned long long b = start[r], e = start[r + 1];
        // stable sort by column: insertion sort for the (already sorted) rows
        // save_matrix_market writes, a merge sort for long unsorted rows
        if (e - b > 64 && !std::is_sorted(cols.begin() + b, cols.begin() + e)) {
            std::vector<std::pair<unsigned long long, double>> row(e - b);
            for (unsigned long long a = b; a < e; ++a) row[a - b] = {cols[a], vals[a]};
            std::stable_sort(row.begin(), row.end(),
                             [](const auto& x, const auto& y) { return x.first < y.first; });
            for (unsigned long long a = b; a < e; ++a) {
                cols[a] = row[a - b].first;
                vals[a] = row[a - b].second;
            }
        }
        for (unsigned long long a = b + 1; a < e; ++a) {
            const unsigned long long c = cols[a];
            const double x = vals[a];
            unsigned long long q = a;
            while (q > b && cols[q - 1] > c) {
                cols[q] = cols[q - 1];
                vals[q] = vals[q - 1];
                --q;
            }
            cols[q] = c;
            vals[q] = x;
        }
        unsigned long long a = b;
        while (a < e) {
            const unsigned long long c = cols[a];
            double s = 0.0;
            while (a < e && cols[a] == c) s += vals[a++];
            if (s != 0.0) {
                ci.push_back(c);
                v.push_back(s);
                ++rp[r + 1];
            }
        }
    }
    for (unsigned long long r = 0; r < dim; ++r) rp[r + 1] += rp[r];
    out->n = dim;
    out->nnz = ci.size();
    out->row_ptr = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (dim + 1)));
    out->col_idx = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * std::max<size_t>(ci.size(), 1)));
    out->values = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(v.size(), 1)));
    if (!out->row_ptr || !out->col_idx || !out->values) {
        nlsp_io_csr_free(out);
        throw std::bad_alloc();
    }
    std::copy(rp.begin(), rp.end(), out->row_ptr);
    std::copy(ci.begin(), ci.end(), out->col_idx);
    std::copy(v.begin(), v.end(), out->values);
}

void load_mm(const std::string& path, nlsp_host_csr* out) {
    std::string buf;
    if (!read_file(path, buf)) throw IoError("cannot open for read: " + path);
    Lines lines{buf};
    std::string line;
    if (!lines.next(line)) throw IoError("empty file: " + path);
    const bool symmetric = line.find("symmetric") != std::string::npos;
    if (line.rfind("%%MatrixMarket", 0) != 0 || line.find("coordinate") == std::string::npos)
        throw IoError("unsupported MatrixMarket header in " + path);
    do {
        if (!lines.next(line)) throw IoError("missing size line: " + path);
    } while (!line.empty() && line[0] == '%');
    Cursor hdr{line.data(), line.data() + line.size()};
    const unsigned long long rows = hdr.u64();
    const unsigned long long cols = hdr.u64();
    const unsigned long long nnz = hdr.u64();
    if (rows != cols) throw IoError("matrix is not square: " + path);
    std::vector<Trip> trip;
    trip.reserve(symmetric ? 2 * std::min<unsigned long long>(nnz, buf.size()) : std::min<unsigned long long>(nnz, buf.size()));
    Cursor in{buf.data() + lines.pos, buf.data() + buf.size()};
    for (unsigned long long k = 0; k < nnz; ++k) {
        const unsigned long long i = in.u64();
        const unsigned long long j = in.u64();
        const double v = in.f64();
        if (in.fail) throw IoError("truncated entries: " + path);
        trip.push_back({i - 1, j - 1, v});
        if (symmetric && i != j) trip.push_back({j - 1, i - 1, v});
    }
    from_triplets(rows, trip, out);
}

void save_mm(const nlsp_host_csr* a, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open for write: " + path);
    unsigned long long count = 0;
    for (unsigned long long i = 0; i < a->n; ++i)
        for (unsigned long long k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
            if (a->col_idx[k] <= i) ++count;
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real symmetric\n");
    std::fprintf(f, "%llu %llu %llu\n", (unsigned long long)a->n, (unsigned long long)a->n, count);
    bool ok = true;
    for (unsigned long long i = 0; i < a->n && ok; ++i)
        for (unsigned long long k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
            if (a->col_idx[k] <= i)
                ok = std::fprintf(f, "%llu %llu %.17g\n", i + 1, (unsigned long long)a->col_idx[k] + 1,
                                  a->values[k]) > 0;
    if (std::fclose(f) != 0 || !ok) throw IoError("write failed: " + path);
}

// --- csv.hpp / Manifest (instance_io.hpp:20-95) -----------------------------
struct Csv {
    std::vector<std::string> header;
    std::vector<std::vector<std::string>> rows;
    size_t column(const std::string& name) const {
        for (size_t i = 0; i < header.size(); ++i)
            if (header[i] == name) return i;
        throw ValidationError("csv: no column named " + name);
    }
};

std::vector<std::string> split_csv_line(const std::string& line) {
    std::vector<std::string> cells;
    std::string cur;
    for (char ch : line) {
        if (ch == ',') {
            cells.push_back(cur);
            cur.clear();
        } else {
            cur.push_back(ch);
        }
    }
    cells.push_back(cur);
    return cells;
}

Csv load_csv(const std::string& path) {
    std::string buf;
    if (!read_file(path, buf)) throw IoError("cannot open for read: " + path);
    Csv t;
    Lines lines{buf};
    std::string line;
    bool have_header = false;
    while (lines.next(line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty() || line[0] == '#') continue;
        if (!have_header) {
            t.header = split_csv_line(line);
            have_header = true;
        } else {
            t.rows.push_back(split_csv_line(line));
        }
    }
    if (!have_header) throw IoError("csv without header: " + path);
    return t;
}

// std::stod: strtod of the whole cell (leading space skipped, trailing text
// ignored); no conversion -> invalid_argument, ERANGE -> out_of_range
double to_double(const std::string& s) {
    const char* b = s.c_str();
    char* e = nullptr;
    errno = 0;
    const double v = std::strtod(b, &e);
    if (e == b) throw std::invalid_argument("stod");
    if (errno == ERANGE) throw std::out_of_range("stod");
    return v;
}

unsigned long long to_u64(const std::string& s) {
    const char* b = s.c_str();
    char* e = nullptr;
    errno = 0;
    const unsigned long long v = std::strtoull(b, &e, 10);
    if (e == b) throw std::invalid_argument("stoull");
    if (errno == ERANGE) throw std::out_of_range("stoull");
    return v;
}

const std::string& cell(const Csv& t, size_t r, size_t c) {
    if (r >= t.rows.size() || c >= t.rows[r].size()) throw std::out_of_range("csv: row too short");
    return t.rows[r][c];
}

struct Manifest {
    std::vector<std::pair<std::string, std::string>> kv;
    const std::string& get(const std::string& key) const {
        for (const auto& e : kv)
            if (e.first == key) return e.second;
        throw ValidationError("manifest: missing key " + key);
    }
    bool has(const std::string& key) const {
        for (const auto& e : kv)
            if (e.first == key) return true;
        return false;
    }
};

Manifest load_manifest(const std::string& path) {
    std::string buf;
    if (!read_file(path, buf)) throw IoError("cannot open for read: " + path);
    Manifest m;
    Lines lines{buf};
    std::string line;
    auto trim = [](const std::string& s) {
        const auto b = s.find_first_not_of(" \t");
        const auto e = s.find_last_not_of(" \t\r");
        return b == std::string::npos ? std::string() : s.substr(b, e - b + 1);
    };
    while (lines.next(line)) {
        if (line.empty() || line[0] == '#') continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw ValidationError("manifest: bad line: " + line);
        const std::string k = trim(line.substr(0, eq)), v = trim(line.substr(eq + 1));
        bool found = false;
        for (auto& e : m.kv)
            if (e.first == k) {
                e.second = v;
                found = true;
            }
        if (!found) m.kv.emplace_back(k, v);
    }
    return m;
}

template <class T>
T* alloc_n(size_t n) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<size_t>(n, 1)));
    if (!p) throw std::bad_alloc();
    return p;
}

void load_instance(const std::string& dir, nlsp_instance* inst) {
    const Manifest m = load_manifest(dir + "/manifest.txt");
    const std::string fam = m.get("family");
    if (fam == "diffusion") inst->family = 0;
    else if (fam == "anisotropic") inst->family = 1;
    else if (fam == "screened_poisson") inst->family = 2;
    else throw ValidationError("unknown PDE family: " + fam);
    inst->grid_n = to_u64(m.get("N"));
    inst->seed = to_u64(m.get("seed"));
    inst->jitter = to_double(m.get("jitter"));

    const Csv vert = load_csv(dir + "/vertices.csv");
    const size_t cx = vert.column("x"), cy = vert.column("y"), cb = vert.column("boundary");
    inst->n_vertices = vert.rows.size();
    inst->vertices = alloc_n<double>(2 * vert.rows.size());
    inst->boundary_mask = alloc_n<uint8_t>(vert.rows.size());
    for (size_t r = 0; r < vert.rows.size(); ++r) {
        inst->vertices[2 * r] = to_double(cell(vert, r, cx));
        inst->vertices[2 * r + 1] = to_double(cell(vert, r, cy));
        inst->boundary_mask[r] = to_double(cell(vert, r, cb)) != 0.0 ? 1 : 0;
    }
    const Csv tri = load_csv(dir + "/triangles.csv");
    const size_t c0 = tri.column("v0"), c1 = tri.column("v1"), c2 = tri.column("v2");
    inst->n_triangles = tri.rows.size();
    inst->triangles = alloc_n<uint64_t>(3 * tri.rows.size());
    for (size_t r = 0; r < tri.rows.size(); ++r) {
        inst->triangles[3 * r] = (uint64_t)to_double(cell(tri, r, c0));
        inst->triangles[3 * r + 1] = (uint64_t)to_double(cell(tri, r, c1));
        inst->triangles[3 * r + 2] = (uint64_t)to_double(cell(tri, r, c2));
    }
    load_mm(dir + "/matrix.mtx", &inst->matrix);
    const Csv rhs = load_csv(dir + "/rhs.csv");
    const size_t cf = rhs.column("f");
    inst->rhs = alloc_n<double>(rhs.rows.size());
    for (size_t r = 0; r < rhs.rows.size(); ++r) inst->rhs[r] = to_double(cell(rhs, r, cf));
    if (rhs.rows.size() != inst->matrix.n)
        throw ValidationError("instance: rhs length does not match the matrix");
    const Csv co = load_csv(dir + "/coefficients.csv");
    std::vector<size_t> cc;
    if (inst->family == 0) cc = {co.column("g")};
    else if (inst->family == 1) cc = {co.column("k11"), co.column("k12"), co.column("k22")};
    else cc = {co.column("kappa")};
    inst->coeff_cols = cc.size();
    inst->coefficients = alloc_n<double>(cc.size() * co.rows.size());
    for (size_t r = 0; r < co.rows.size(); ++r)
        for (size_t q = 0; q < cc.size(); ++q) inst->coefficients[r * cc.size() + q] = to_double(cell(co, r, cc[q]));
    inst->alpha = inst->family == 2 ? to_double(m.get("alpha")) : 0.0;
}

// --- MlpModel checkpoints and initialisation (mlp.hpp:57-88, 255-303) -------
uint64_t mlp_param_count(const std::vector<uint64_t>& w) {
    if (w.size() < 2) throw ValidationError("mlp: need at least input and output widths");
    uint64_t total = 0;
    for (size_t l = 0; l + 1 < w.size(); ++l) {
        total += w[l] * w[l + 1] + w[l + 1];
        if (l + 2 < w.size()) total += 2 * w[l + 1];
    }
    return total;
}

void mlp_fill(nlsp_host_mlp* out, const std::vector<uint64_t>& w, uint64_t np, const std::string& manifest) {
    out->nwidths = w.size();
    out->widths = alloc_n<uint64_t>(w.size());
    std::copy(w.begin(), w.end(), out->widths);
    out->nparams = np;
    out->params = alloc_n<double>(np);
    out->manifest = alloc_n<char>(manifest.size() + 1);
    std::memcpy(out->manifest, manifest.c_str(), manifest.size() + 1);
}

void mlp_load(const std::string& path, nlsp_host_mlp* out) {
    std::string buf;
    if (!read_file(path, buf)) throw IoError("cannot open for read: " + path);
    size_t pos = 0;
    bool ok = true;
    auto get = [&](void* dst, size_t bytes) {
        if (pos + bytes > buf.size()) {
            ok = false;
            const size_t have = pos < buf.size() ? buf.size() - pos : 0;
            std::memset(dst, 0, bytes);
            if (have) std::memcpy(dst, buf.data() + pos, have);
            pos = buf.size();
            return;
        }
        std::memcpy(dst, buf.data() + pos, bytes);
        pos += bytes;
    };
    auto get_u64 = [&]() {
        uint64_t v = 0;
        get(&v, 8);
        return v;
    };
    char magic[8] = {};
    get(magic, 8);
    if (!ok || std::string(magic, 8) != "NLSPCKP1") throw IoError("bad checkpoint magic: " + path);
    const uint64_t nw = get_u64();
    if (!ok || nw > (buf.size() / 8)) throw IoError("truncated checkpoint: " + path);
    std::vector<uint64_t> w(nw);
    for (auto& x : w) x = get_u64();
    const uint64_t expect = mlp_param_count(w);  // ValidationError for < 2 widths (the ctor's)
    const uint64_t np = get_u64();
    if (np != expect) throw IoError("checkpoint parameter count mismatch: " + path);
    if (np > buf.size() / 8) throw IoError("truncated checkpoint: " + path);
    mlp_fill(out, w, np, "");
    get(out->params, 8 * np);
    pos += 16 * np;  // Adam m, v (not kept)
    if (pos > buf.size()) {
        ok = false;
        pos = buf.size();
    }
    (void)get_u64();  // adam step
    const uint64_t mlen = get_u64();
    if (!ok || mlen > buf.size() - pos) throw IoError("truncated checkpoint: " + path);
    std::free(out->manifest);
    out->manifest = alloc_n<char>(mlen + 1);
    std::memcpy(out->manifest, buf.data() + pos, mlen);
    out->manifest[mlen] = '\0';
}

void mlp_save(const nlsp_host_mlp* m, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open for write: " + path);
    bool ok = std::fwrite("NLSPCKP1", 1, 8, f) == 8;
    auto put = [&](const void* p, size_t bytes) { ok = ok && std::fwrite(p, 1, bytes, f) == bytes; };
    auto put_u64 = [&](uint64_t v) { put(&v, 8); };
    put_u64(m->nwidths);
    for (uint64_t l = 0; l < m->nwidths; ++l) put_u64(m->widths[l]);
    put_u64(m->nparams);
    put(m->params, 8 * m->nparams);
    std::vector<double> zeros(std::min<uint64_t>(m->nparams, 1 << 20), 0.0);
    for (int rep = 0; rep < 2; ++rep)
        for (uint64_t done = 0; done < m->nparams;) {
            const uint64_t c = std::min<uint64_t>(zeros.size(), m->nparams - done);
            put(zeros.data(), 8 * c);
            done += c;
        }
    put_u64(0);
    const size_t mlen = m->manifest ? std::strlen(m->manifest) : 0;
    put_u64(mlen);
    if (mlen) put(m->manifest, mlen);
    if (std::fclose(f) != 0 || !ok) throw IoError("write failed: " + path);
}

void mlp_init(const uint64_t* widths, uint64_t nw, uint64_t seed, nlsp_host_mlp* out) {
    std::vector<uint64_t> w(widths, widths + nw);
    const uint64_t np = mlp_param_count(w);
    mlp_fill(out, w, np, "");
    std::fill(out->params, out->params + np, 0.0);
    // one Rng(mix_seed(seed, 0x6d6c70)) stream across the layers' weights, in order
    uint64_t nweights = 0;
    for (size_t l = 0; l + 1 < w.size(); ++l) nweights += w[l] * w[l + 1];
    std::vector<double> z(nweights);
    nlsp_host::normal_stream(nlsp_host::mix_seed(seed, 0x6d6c70), nweights, z.data());
    uint64_t off = 0, zi = 0;
    for (size_t l = 0; l + 1 < w.size(); ++l) {
        const uint64_t fi = w[l], fo = w[l + 1];
        const double sd = std::sqrt(2.0 / static_cast<double>(fi));
        for (uint64_t i = 0; i < fi * fo; ++i) out->params[off + i] = 0.0 + sd * z[zi++];  // normal(0, sd)
        off += fi * fo + fo;
        if (l + 2 < w.size()) {
            for (uint64_t i = 0; i < fo; ++i) out->params[off + i] = 1.0;  // gain
            off += 2 * fo;
        }
    }
}

}  // namespace

extern "C" {

int nlsp_io_load_matrix_market(const char* path, nlsp_host_csr* out) {
    if (!path || !out) {
        g_err = "load_matrix_market: null argument";
        return NLSP_IO_E_VALIDATION;
    }
    *out = nlsp_host_csr{};
    return guarded([&] { load_mm(path, out); });
}

int nlsp_io_save_matrix_market(const nlsp_host_csr* a, const char* path) {
    if (!path || !a || !a->row_ptr) {
        g_err = "save_matrix_market: null argument";
        return NLSP_IO_E_VALIDATION;
    }
    return guarded([&] { save_mm(a, path); });
}

void nlsp_io_csr_free(nlsp_host_csr* a) {
    if (!a) return;
    std::free(a->row_ptr);
    std::free(a->col_idx);
    std::free(a->values);
    a->row_ptr = a->col_idx = nullptr;
    a->values = nullptr;
}

int nlsp_io_load_instance(const char* dir, nlsp_instance* out) {
    if (!dir || !out) {
        g_err = "load_instance: null argument";
        return NLSP_IO_E_VALIDATION;
    }
    *out = nlsp_instance{};
    const int st = guarded([&] { load_instance(dir, out); });
    if (st) nlsp_io_instance_free(out);
    return st;
}

void nlsp_io_instance_free(nlsp_instance* inst) {
    if (!inst) return;
    nlsp_io_csr_free(&inst->matrix);
    std::free(inst->rhs);
    std::free(inst->vertices);
    std::free(inst->boundary_mask);
    std::free(inst->triangles);
    std::free(inst->coefficients);
    inst->rhs = inst->vertices = inst->coefficients = nullptr;
    inst->boundary_mask = nullptr;
    inst->triangles = nullptr;
}

int nlsp_io_mlp_load(const char* path, nlsp_host_mlp* out) {
    if (!path || !out) {
        g_err = "mlp load: null argument";
        return NLSP_IO_E_VALIDATION;
    }
    *out = nlsp_host_mlp{};
    const int st = guarded([&] { mlp_load(path, out); });
    if (st) nlsp_io_mlp_free(out);
    return st;
}

int nlsp_io_mlp_save(const nlsp_host_mlp* m, const char* path) {
    if (!path || !m || !m->widths || !m->params) {
        g_err = "mlp save: null argument";
        return NLSP_IO_E_VALIDATION;
    }
    return guarded([&] { mlp_save(m, path); });
}

int nlsp_io_mlp_init(const uint64_t* widths, uint64_t nwidths, uint64_t seed, nlsp_host_mlp* out) {
    if (!widths || !out) {
        g_err = "mlp init: null argument";
        return NLSP_IO_E_VALIDATION;
    }
    *out = nlsp_host_mlp{};
    const int st = guarded([&] { mlp_init(widths, nwidths, seed, out); });
    if (st) nlsp_io_mlp_free(out);
    return st;
}

void nlsp_io_mlp_free(nlsp_host_mlp* m) {
    if (!m) return;
    std::free(m->widths);
    std::free(m->params);
    std::free(m->manifest);
    *m = nlsp_host_mlp{};
}

const char* nlsp_io_last_error(void) { return g_err.c_str(); }

}  // extern "C"
