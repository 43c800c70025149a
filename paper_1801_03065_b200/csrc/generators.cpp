// Host-side input generators for the BASELINE.json configurations (bench and
// test plumbing, not the hot path).  One generator is shared by the GPU path
// and the CPU oracle so both see byte-identical CSR buffers.
// Definitions follow SURVEY.md Appendix A exactly, including the RNG draw
// order, so the structural counts of §8d reproduce:
//   laplace2d   5-point, row r = x*n + y, neighbours (-1,0),(0,-1),(0,0),(0,1),(1,0)
//   laplace3d   27-point, row r = (x*n + y)*n + z, offsets dx,dy,dz in lexicographic order
//   rmat        Graph500 R-MAT (a,b,c,d) = (.57,.19,.19,.05), no label permutation,
//               duplicates summed in encounter order (build_csr semantics,
//               csr_matrix.cpp:18-80), self loops kept, vals U(-1,1)
//   aggregation piecewise-constant 2x2x2 aggregation prolongator P (1 nnz/row, value 1)
// Stencil weights are perturbed w*(1 + eps*U(-1,1)) from mt19937_64(seed) in CSR
// order so the 1e-12 value check has power (SURVEY.md §8c caveat).
//
// kkg_read_mm: MatrixMarket ingest (a chunked multi-threaded tokeniser, see
// read_mm below), entries through the same build_csr semantics (duplicates
// summed in encounter order).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <climits>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

namespace {

struct Mat {
    int32_t rows = 0, cols = 0;
    std::vector<int64_t> rowptr;
    std::vector<int32_t> ci;
    std::vector<double> v;
};

void perturb(Mat& m, double eps, uint64_t seed)
{
    if (eps == 0.0)
        return;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (double& x : m.v)
        x = x * (1.0 + eps * u(rng));
}

// build_csr semantics: counting sort by row (stable), stable sort by column,
// duplicates summed in encounter order.
Mat build(int32_t rows, int32_t cols, const std::vector<int32_t>& r, const std::vector<int32_t>& c,
          const std::vector<double>& v)
{
    Mat m;
    m.rows = rows;
    m.cols = cols;
    std::vector<int64_t> cnt(static_cast<size_t>(rows) + 1, 0);
    for (int32_t x : r)
        ++cnt[static_cast<size_t>(x) + 1];
    for (int32_t i = 0; i < rows; ++i)
        cnt[i + 1] += cnt[i];
    std::vector<int32_t> sc(r.size());
    std::vector<double> sv(r.size());
    {
        std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
        for (size_t q = 0; q < r.size(); ++q) {
            const int64_t p = fill[r[q]]++;
            sc[p] = c[q];
            sv[p] = v[q];
        }
    }
    m.rowptr.assign(static_cast<size_t>(rows) + 1, 0);
    m.ci.reserve(r.size());
    m.v.reserve(r.size());
    std::vector<int64_t> perm;
    for (int32_t i = 0; i < rows; ++i) {
        const int64_t lo = cnt[i], hi = cnt[i + 1];
        perm.resize(hi - lo);
        std::iota(perm.begin(), perm.end(), lo);
        std::stable_sort(perm.begin(), perm.end(), [&](int64_t x, int64_t y) { return sc[x] < sc[y]; });
        for (size_t q = 0; q < perm.size(); ++q) {
            if (q > 0 && sc[perm[q - 1]] == sc[perm[q]])
                m.v.back() += sv[perm[q]];
            else {
                m.ci.push_back(sc[perm[q]]);
                m.v.push_back(sv[perm[q]]);
            }
        }
        m.rowptr[i + 1] = static_cast<int64_t>(m.ci.size());
    }
    return m;
}

// ---- MatrixMarket ingest ------------------------------------------------------
// The whole file is read into one buffer; the entry section is cut at line
// boundaries into one slice per host thread, each slice is tokenised in place
// (no per-line strings, no iostreams), and the slices' triplets are spliced in
// file order before build() — so the result is identical to a sequential
// read.  Contract kept from the reference reader (matrix_market.cpp:48-132):
// coordinate matrices only; real, integer or pattern fields; general or
// symmetric (off-diagonal entries mirrored); 1-based indices checked against
// the size line; '%' lines and blank lines skipped anywhere; exactly the
// declared number of entries is read (anything after them is ignored); every
// malformed input is an error carrying its 1-based line number.
struct MmError {
    std::string what;
    long line;
};

struct Cursor {
    const char* p;
    const char* end;
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

// next line [*b, *e) (without the newline); false at end of buffer
inline bool next_line(Cursor& c, const char** b, const char** e)
{
    if (c.p >= c.end)
        return false;
    const char* nl = static_cast<const char*>(std::memchr(c.p, '\n', static_cast<size_t>(c.end - c.p)));
    *b = c.p;
    *e = nl ? nl : c.end;
    c.p = nl ? nl + 1 : c.end;
    return true;
}

// comment or whitespace-only line
inline bool skip_line(const char* b, const char* e)
{
    while (b < e && is_space(*b))
        ++b;
    return b == e || *b == '%';
}

inline const char* skip_ws(const char* p, const char* e)
{
    while (p < e && is_space(*p))
        ++p;
    return p;
}

// unsigned/signed decimal integer token; false if none or out of int64 range
inline bool parse_i64(const char*& p, const char* e, long long* out)
{
    p = skip_ws(p, e);
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-'))
        neg = *p++ == '-';
    const char* d0 = p;
    unsigned long long v = 0;
    while (p < e && *p >= '0' && *p <= '9') {
        const unsigned digit = static_cast<unsigned>(*p - '0');
        if (v > (ULLONG_MAX - digit) / 10)
            return false;
        v = v * 10 + digit;
        ++p;
    }
    if (p == d0 || v > static_cast<unsigned long long>(LLONG_MAX))
        return false;
    *out = neg ? -static_cast<long long>(v) : static_cast<long long>(v);
    return p == e || is_space(*p);
}

inline bool parse_f64(const char*& p, const char* e, double* out)
{
    p = skip_ws(p, e);
    if (p == e)
        return false;
    // strtod needs a terminator: copy the token (values are short)
    char tok[128];
    size_t n = 0;
    while (p < e && !is_space(*p) && n + 1 < sizeof(tok))
        tok[n++] = *p++;
    tok[n] = 0;
    char* stop = nullptr;
    *out = std::strtod(tok, &stop);
    return stop != tok && *stop == 0;
}

std::string lower(std::string x)
{
    for (char& ch : x)
        ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return x;
}

struct Slice {
    const char* b;
    const char* e;
    long long first_line = 0; // 1-based line number of the slice's first line
    std::vector<int32_t> r, c;
    std::vector<double> v;
    long long entries = 0;        // entry lines parsed
    long long err_at = -1;        // entries parsed before the first bad line
    long long err_line = 0;       // line number of that bad line (slice-relative, 0-based)
    std::string err;
};

void parse_slice(Slice& s, long long rows, long long cols, bool pattern, bool symmetric)
{
    Cursor c{s.b, s.e};
    const char *lb, *le;
    long long ln = -1;
    while (next_line(c, &lb, &le)) {
        ++ln;
        if (skip_line(lb, le))
            continue;
        const char* p = lb;
        long long ri = 0, ci = 0;
        double x = 1.0;
        const char* bad = nullptr;
        if (!parse_i64(p, le, &ri) || !parse_i64(p, le, &ci))
            bad = "malformed entry indices";
        else if (ri < 1 || ri > rows || ci < 1 || ci > cols)
            bad = "entry index outside the declared size";
        else if (!pattern && !parse_f64(p, le, &x))
            bad = "malformed entry value";
        if (bad) {
            s.err_at = s.entries;
            s.err_line = ln;
            s.err = bad;
            return;
        }
        s.r.push_back(static_cast<int32_t>(ri - 1));
        s.c.push_back(static_cast<int32_t>(ci - 1));
        s.v.push_back(x);
        if (symmetric && ri != ci) {
            s.r.push_back(static_cast<int32_t>(ci - 1));
            s.c.push_back(static_cast<int32_t>(ri - 1));
            s.v.push_back(x);
        }
        ++s.entries;
    }
}

Mat read_mm(const char* path)
{
    std::FILE* f = std::fopen(path, "rb");
    if (!f)
        throw MmError{std::string("MatrixMarket: cannot read ") + path, 0};
    std::string buf;
    {
        char tmp[1 << 16];
        size_t got;
        while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0)
            buf.append(tmp, got);
        std::fclose(f);
    }
    Cursor cur{buf.data(), buf.data() + buf.size()};
    const char *lb, *le;
    long long line = 0;
    // banner: %%MatrixMarket matrix coordinate <field> <symmetry>
    if (!next_line(cur, &lb, &le))
        throw MmError{"MatrixMarket: empty file", 1};
    ++line;
    std::vector<std::string> words;
    for (const char* p = lb; p < le;) {
        p = skip_ws(p, le);
        const char* q = p;
        while (q < le && !is_space(*q))
            ++q;
        if (q > p)
            words.emplace_back(p, q);
        p = q;
    }
    if (words.size() < 5 || words[0] != "%%MatrixMarket" || lower(words[1]) != "matrix")
        throw MmError{"MatrixMarket: first line is not a matrix banner", line};
    if (lower(words[2]) != "coordinate")
        throw MmError{"MatrixMarket: '" + words[2] + "' storage is not supported (coordinate only)", line};
    const std::string field = lower(words[3]), symmetry = lower(words[4]);
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer")
        throw MmError{"MatrixMarket: field '" + words[3] + "' is not supported", line};
    const bool symmetric = symmetry == "symmetric";
    if (!symmetric && symmetry != "general")
        throw MmError{"MatrixMarket: symmetry '" + words[4] + "' is not supported", line};
    // size line: the first non-comment, non-blank line
    long long rows = -1, cols = -1, entries = -1;
    for (;;) {
        if (!next_line(cur, &lb, &le))
            throw MmError{"MatrixMarket: no size line", line + 1};
        ++line;
        if (skip_line(lb, le))
            continue;
        const char* p = lb;
        if (!parse_i64(p, le, &rows) || !parse_i64(p, le, &cols) || !parse_i64(p, le, &entries))
            throw MmError{"MatrixMarket: size line needs rows, columns and entries", line};
        break;
    }
    if (rows < 0 || cols < 0 || entries < 0)
        throw MmError{"MatrixMarket: negative size", line};
    const long long lim = std::numeric_limits<int32_t>::max();
    if (rows > lim || cols > lim || entries > lim)
        throw MmError{"MatrixMarket: size beyond the 32-bit index type", line};

    // slices of the entry section at line boundaries
    const char* body = cur.p;
    const size_t len = static_cast<size_t>(cur.end - body);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nsl = std::max<size_t>(1, std::min<size_t>(hw, len / (1 << 20)));
    std::vector<Slice> sl(nsl);
    const char* at = body;
    for (size_t t = 0; t < nsl; ++t) {
        const char* stop = t + 1 == nsl ? cur.end : body + len * (t + 1) / nsl;
        if (stop < at)
            stop = at;
        if (t + 1 < nsl) {
            const char* nl = static_cast<const char*>(std::memchr(stop, '\n', static_cast<size_t>(cur.end - stop)));
            stop = nl ? nl + 1 : cur.end;
        }
        sl[t].b = at;
        sl[t].e = stop;
        at = stop;
    }
    {
        std::vector<std::thread> th;
        for (size_t t = 1; t < nsl; ++t)
            th.emplace_back(parse_slice, std::ref(sl[t]), rows, cols, pattern, symmetric);
        parse_slice(sl[0], rows, cols, pattern, symmetric);
        for (auto& x : th)
            x.join();
    }
    // splice in file order; only the first `entries` entries count, so an
    // error after them is ignored
    long long taken = 0, line0 = line + 1;
    std::vector<int32_t> r, c;
    std::vector<double> v;
    r.reserve(static_cast<size_t>(symmetric ? 2 * entries : entries));
    c.reserve(r.capacity());
    v.reserve(r.capacity());
    for (Slice& s : sl) {
        const long long lines_in = static_cast<long long>(std::count(s.b, s.e, '\n'));
        if (taken < entries) {
            if (s.err_at >= 0 && taken + s.err_at < entries)
                throw MmError{"MatrixMarket: " + s.err, line0 + s.err_line};
            // triplets of this slice up to the entry limit (symmetric entries
            // contribute one or two triplets)
            size_t q = 0;
            for (long long k = 0; k < s.entries && taken < entries; ++k, ++taken) {
                const size_t w = symmetric && s.r[q] != s.c[q] ? 2 : 1; // an off-diagonal entry and its mirror
                for (size_t u = 0; u < w; ++u, ++q) {
                    r.push_back(s.r[q]);
                    c.push_back(s.c[q]);
                    v.push_back(s.v[q]);
                }
            }
        }
        line0 += lines_in;
    }
    if (taken < entries)
        throw MmError{"MatrixMarket: file ends after " + std::to_string(taken) + " of " + std::to_string(entries)
                          + " entries",
                      line0};
    return build(static_cast<int32_t>(rows), static_cast<int32_t>(cols), r, c, v);
}

} // namespace

extern "C" {

// MatrixMarket ingest; NULL on error with the message (and 1-based line, 0 if
// none) in err[0..errlen)
void* kkg_read_mm(const char* path, char* err, int32_t errlen)
{
    try {
        return new Mat(read_mm(path));
    } catch (const MmError& e) {
        const std::string msg = e.line > 0 ? e.what + " (line " + std::to_string(e.line) + ")" : e.what;
        if (err && errlen > 0) {
            std::strncpy(err, msg.c_str(), static_cast<size_t>(errlen) - 1);
            err[errlen - 1] = 0;
        }
        return nullptr;
    }
}

void* kkg_laplace2d(int32_t n, double eps, uint64_t seed)
{
    auto* m = new Mat;
    const int64_t N = int64_t{n} * n;
    m->rows = m->cols = static_cast<int32_t>(N);
    m->rowptr.reserve(N + 1);
    m->rowptr.push_back(0);
    m->ci.reserve(5 * N);
    m->v.reserve(5 * N);
    const int dx[5] = {-1, 0, 0, 0, 1}, dy[5] = {0, -1, 0, 1, 0};
    for (int32_t x = 0; x < n; ++x)
        for (int32_t y = 0; y < n; ++y) {
            for (int q = 0; q < 5; ++q) {
                const int32_t xx = x + dx[q], yy = y + dy[q];
                if (xx < 0 || yy < 0 || xx >= n || yy >= n)
                    continue;
                m->ci.push_back(xx * n + yy);
                m->v.push_back(q == 2 ? 4.0 : -1.0);
            }
            m->rowptr.push_back(static_cast<int64_t>(m->ci.size()));
        }
    perturb(*m, eps, seed);
    return m;
}

void* kkg_laplace3d(int32_t n, double eps, uint64_t seed)
{
    auto* m = new Mat;
    const int64_t N = int64_t{n} * n * n;
    m->rows = m->cols = static_cast<int32_t>(N);
    const int64_t nnz = int64_t(3 * n - 2) * (3 * n - 2) * (3 * n - 2);
    m->rowptr.reserve(N + 1);
    m->rowptr.push_back(0);
    m->ci.reserve(nnz);
    m->v.reserve(nnz);
    for (int32_t x = 0; x < n; ++x)
        for (int32_t y = 0; y < n; ++y)
            for (int32_t z = 0; z < n; ++z) {
                for (int ddx = -1; ddx <= 1; ++ddx)
                    for (int ddy = -1; ddy <= 1; ++ddy)
                        for (int ddz = -1; ddz <= 1; ++ddz) {
                            const int32_t xx = x + ddx, yy = y + ddy, zz = z + ddz;
                            if (xx < 0 || yy < 0 || zz < 0 || xx >= n || yy >= n || zz >= n)
                                continue;
                            m->ci.push_back((xx * n + yy) * n + zz);
                            m->v.push_back(ddx == 0 && ddy == 0 && ddz == 0 ? 26.0 : -1.0);
                        }
                m->rowptr.push_back(static_cast<int64_t>(m->ci.size()));
            }
    perturb(*m, eps, seed);
    return m;
}

void* kkg_rmat(int32_t scale, int32_t edge_factor, uint64_t seed)
{
    const int32_t nv = int32_t{1} << scale;
    const int64_t ne = int64_t{edge_factor} * nv;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0), val(-1.0, 1.0);
    std::vector<int32_t> r(ne), c(ne);
    std::vector<double> v(ne);
    for (int64_t e = 0; e < ne; ++e) {
        int32_t rr = 0, cc = 0;
        for (int32_t l = 0; l < scale; ++l) {
            const double p = u(rng);
            const int q = p < 0.57 ? 0 : p < 0.76 ? 1 : p < 0.95 ? 2 : 3;
            rr = (rr << 1) | (q >> 1);
            cc = (cc << 1) | (q & 1);
        }
        r[e] = rr;
        c[e] = cc;
        v[e] = val(rng);
    }
    return new Mat(build(nv, nv, r, c, v));
}

void* kkg_aggregation(int32_t n)
{
    const int32_t nc = (n + 1) / 2;
    const int64_t N = int64_t{n} * n * n;
    std::vector<int32_t> r(N), c(N);
    std::vector<double> v(N, 1.0);
    for (int32_t x = 0; x < n; ++x)
        for (int32_t y = 0; y < n; ++y)
            for (int32_t z = 0; z < n; ++z) {
                const int64_t row = (int64_t(x) * n + y) * n + z;
                r[row] = static_cast<int32_t>(row);
                c[row] = ((x / 2) * nc + y / 2) * nc + z / 2;
            }
    return new Mat(build(static_cast<int32_t>(N), nc * nc * nc, r, c, v));
}

// transpose (csr_matrix.cpp:82-108 semantics: counting sort, rows come out sorted)
void* kkg_transpose(const void* mp)
{
    const auto& m = *static_cast<const Mat*>(mp);
    auto* t = new Mat;
    t->rows = m.cols;
    t->cols = m.rows;
    t->rowptr.assign(static_cast<size_t>(t->rows) + 1, 0);
    t->ci.resize(m.ci.size());
    t->v.resize(m.v.size());
    for (int32_t c : m.ci)
        ++t->rowptr[static_cast<size_t>(c) + 1];
    for (int32_t i = 0; i < t->rows; ++i)
        t->rowptr[i + 1] += t->rowptr[i];
    std::vector<int64_t> fill(t->rowptr.begin(), t->rowptr.end() - 1);
    for (int32_t i = 0; i < m.rows; ++i)
        for (int64_t p = m.rowptr[i]; p < m.rowptr[i + 1]; ++p) {
            const int64_t q = fill[m.ci[p]]++;
            t->ci[q] = i;
            t->v[q] = m.v[p];
        }
    return t;
}

void kkg_shape(const void* mp, int32_t* rows, int32_t* cols, int64_t* nnz)
{
    const auto& m = *static_cast<const Mat*>(mp);
    *rows = m.rows;
    *cols = m.cols;
    *nnz = static_cast<int64_t>(m.ci.size());
}

void kkg_export(const void* mp, int64_t* rowptr, int32_t* ci, double* v)
{
    const auto& m = *static_cast<const Mat*>(mp);
    std::memcpy(rowptr, m.rowptr.data(), sizeof(int64_t) * m.rowptr.size());
    std::memcpy(ci, m.ci.data(), sizeof(int32_t) * m.ci.size());
    std::memcpy(v, m.v.data(), sizeof(double) * m.v.size());
}

void kkg_free(void* mp) { delete static_cast<Mat*>(mp); }

} // extern "C"
