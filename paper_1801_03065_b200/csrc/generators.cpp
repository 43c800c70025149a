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
// kkg_read_mm: MatrixMarket ingest with the reference reader's contract
// (matrix_market.cpp:48-132): coordinate real/integer/pattern, general or
// symmetric (mirrored off-diagonal entries), 1-based indices checked against
// the size line, '%' comment and blank lines skipped, entries through the
// same build_csr semantics (duplicates summed in encounter order).
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <numeric>
#include <random>
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

bool blank(const std::string& s)
{
    for (char c : s)
        if (c != ' ' && c != '\t' && c != '\r' && c != '\n' && c != '\f' && c != '\v')
            return false;
    return true;
}

struct MmError {
    std::string what;
    long line;
};

long long mm_int(const char*& p, long line, const char* what)
{
    errno = 0;
    char* end = nullptr;
    const long long v = std::strtoll(p, &end, 10);
    if (end == p || errno == ERANGE)
        throw MmError{std::string("expected ") + what, line};
    p = end;
    return v;
}

Mat read_mm(const char* path)
{
    std::ifstream in(path);
    if (!in)
        throw MmError{std::string("cannot open '") + path + "' for reading", 0};
    std::string ln;
    long line = 0;
    if (!std::getline(in, ln))
        throw MmError{"missing MatrixMarket header", 1};
    ++line;
    std::istringstream hdr(ln);
    std::string banner, object, format, field, symmetry;
    hdr >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket" || object != "matrix")
        throw MmError{"not a MatrixMarket matrix header", line};
    if (format != "coordinate")
        throw MmError{"only coordinate format is supported", line};
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer")
        throw MmError{"unsupported field '" + field + "'", line};
    const bool symmetric = symmetry == "symmetric";
    if (!symmetric && symmetry != "general")
        throw MmError{"unsupported symmetry '" + symmetry + "'", line};
    long long rows = 0, cols = 0, entries = 0;
    for (;;) {
        if (!std::getline(in, ln))
            throw MmError{"missing size line", line + 1};
        ++line;
        if ((!ln.empty() && ln[0] == '%') || blank(ln))
            continue;
        const char* p = ln.c_str();
        rows = mm_int(p, line, "row count");
        cols = mm_int(p, line, "column count");
        entries = mm_int(p, line, "entry count");
        break;
    }
    if (rows < 0 || cols < 0 || entries < 0)
        throw MmError{"negative size field", line};
    const long long imax = std::numeric_limits<int32_t>::max();
    if (rows > imax || cols > imax || entries > imax)
        throw MmError{"size exceeds 32-bit index range", line};
    std::vector<int32_t> r, c;
    std::vector<double> v;
    r.reserve(static_cast<size_t>(symmetric ? 2 * entries : entries));
    c.reserve(r.capacity());
    v.reserve(r.capacity());
    for (long long seen = 0; seen < entries;) {
        if (!std::getline(in, ln))
            throw MmError{"unexpected end of file: " + std::to_string(entries - seen) + " entries missing", line + 1};
        ++line;
        if ((!ln.empty() && ln[0] == '%') || blank(ln))
            continue;
        const char* p = ln.c_str();
        const long long ri = mm_int(p, line, "row index");
        const long long ci = mm_int(p, line, "column index");
        if (ri < 1 || ri > rows || ci < 1 || ci > cols)
            throw MmError{"index out of range", line};
        double x = 1.0;
        if (!pattern) {
            char* end = nullptr;
            x = std::strtod(p, &end);
            if (end == p)
                throw MmError{"expected a numeric value", line};
        }
        r.push_back(static_cast<int32_t>(ri - 1));
        c.push_back(static_cast<int32_t>(ci - 1));
        v.push_back(x);
        if (symmetric && ri != ci) {
            r.push_back(static_cast<int32_t>(ci - 1));
            c.push_back(static_cast<int32_t>(ri - 1));
            v.push_back(x);
        }
        ++seen;
    }
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
