// cvk_mmio.cu -- Matrix Market coordinate complex general I/O at scale
// (SURVEY.md 8(f) rank 2), host code.
//
// Same results as the reference's read_matrix_market + csr_from_triplets
// (mmio.cpp:28-63, numkit.cpp:41-75): 1-based entries, duplicates summed in
// input order, columns sorted per row, values parsed with strtod (correctly
// rounded, as iostream >> double); the writer prints "%.17g" like
// std::setprecision(17) (mmio.cpp:10-21), byte for byte.
//
// The reference reader holds a 32 B/nnz triplet vector, copies it into
// csr_from_triplets and stable-sorts it: >= 48 GB of host RAM at 7.5e8 nnz.
// Here the file is mapped, the entry lines are parsed by T threads (strtod
// in parallel), a counting sort by row keeps input order (stable), and rows
// are sorted and merged in parallel -- about 56 B/nnz at peak.  Text after
// the nnz-th entry must still be entries (the reference stops reading).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cavac_b200.h"

int cvk_fail(int code, const std::string& msg);

namespace {

struct Mapped {
    const char* p = nullptr;
    size_t n = 0;
    int fd = -1;
    ~Mapped() {
        if (p && n) munmap((void*)p, n);
        if (fd >= 0) close(fd);
    }
};

int nthreads_for(int want) {
    int t = want > 0 ? want : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(t, 256));
}

// one entry line: "r c re im" (any whitespace); false on a malformed entry
bool parse_entry(const char*& s, const char* e, uint64_t& r, uint64_t& c, double& re, double& im) {
    auto skip = [&]() {
        while (s < e && (*s == ' ' || *s == '\t' || *s == '\n' || *s == '\r')) ++s;
    };
    auto num_u = [&](uint64_t& v) {
        skip();
        if (s >= e || *s < '0' || *s > '9') return false;
        char* end = nullptr;
        errno = 0;
        v = std::strtoull(s, &end, 10);
        if (errno || end == s) return false;
        s = end;
        return true;
    };
    auto num_d = [&](double& v) {
        skip();
        if (s >= e) return false;
        char* end = nullptr;
        v = std::strtod(s, &end);  // the buffer ends in whitespace (see cvk_mm_read)
        if (end == s) return false;
        s = end;
        return true;
    };
    return num_u(r) && num_u(c) && num_d(re) && num_d(im);
}

}  // namespace

extern "C" int cvk_mm_read(const char* path, int nthreads, cvk_mm_matrix* out) {
    if (!path || !out) return cvk_fail(CVK_EINVAL, "cvk_mm_read: null argument");
    std::memset(out, 0, sizeof(*out));
    Mapped m;
    m.fd = open(path, O_RDONLY);
    if (m.fd < 0) return cvk_fail(CVK_EINVAL, std::string("cannot open ") + path);
    struct stat sb;
    if (fstat(m.fd, &sb) != 0) return cvk_fail(CVK_EINVAL, std::string("cannot open ") + path);
    m.n = (size_t)sb.st_size;
    if (m.n == 0) return cvk_fail(CVK_EINVAL, "matrix market: empty stream");
    void* mp = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
    if (mp == MAP_FAILED) return cvk_fail(CVK_EINVAL, std::string("cannot map ") + path);
    m.p = (const char*)mp;
    // strtod must not run past the mapping: a file whose last byte is not
    // whitespace is read into a buffer with a newline appended
    std::vector<char> copy;
    const char* s = m.p;
    const char* e = m.p + m.n;
    const char last = m.p[m.n - 1];
    if (last != '\n' && last != ' ' && last != '\t' && last != '\r') {
        copy.assign(m.p, m.p + m.n);
        copy.push_back('\n');
        s = copy.data();
        e = copy.data() + copy.size();
    }
    auto next_line = [&](const char*& a) -> std::string {
        const char* b = a;
        while (a < e && *a != '\n') ++a;
        std::string l(b, a);
        if (a < e) ++a;
        if (!l.empty() && l.back() == '\r') l.pop_back();
        return l;
    };
    // header (mmio.cpp:29-44)
    const std::string hdr = next_line(s);
    if (hdr.rfind("%%MatrixMarket", 0) != 0) return cvk_fail(CVK_EINVAL, "matrix market: missing header");
    {
        char tag[64] = {0}, obj[64] = {0}, fmt[64] = {0}, field[64] = {0}, symm[64] = {0};
        std::sscanf(hdr.c_str(), "%63s %63s %63s %63s %63s", tag, obj, fmt, field, symm);
        if (std::strcmp(obj, "matrix") || std::strcmp(fmt, "coordinate") || std::strcmp(field, "complex") ||
            std::strcmp(symm, "general"))
            return cvk_fail(CVK_EINVAL, "matrix market: unsupported header \"" + hdr + "\"");
    }
    // comment / empty lines, then the size line (mmio.cpp:45-51)
    std::string line;
    for (;;) {
        if (s >= e) return cvk_fail(CVK_EINVAL, "matrix market: bad size line");
        line = next_line(s);
        if (!line.empty() && line[0] != '%') break;
    }
    unsigned long long nr = 0, nc = 0, nz = 0;
    if (std::sscanf(line.c_str(), "%llu %llu %llu", &nr, &nc, &nz) != 3)
        return cvk_fail(CVK_EINVAL, "matrix market: bad size line");
    const int64_t nrows = (int64_t)nr, ncols = (int64_t)nc, nnz_in = (int64_t)nz;

    // split the entry block at line ends; each thread parses its lines
    const int T = nthreads_for(nthreads);
    std::vector<const char*> cut(T + 1);
    cut[0] = s;
    cut[T] = e;
    for (int t = 1; t < T; ++t) {
        const char* q = s + (size_t)(e - s) * t / T;
        if (q < cut[t - 1]) q = cut[t - 1];
        while (q < e && *q != '\n') ++q;
        cut[t] = q < e ? q + 1 : e;
    }
    struct Part {
        std::vector<int64_t> r, c;
        std::vector<double> v;  // re, im
        int err = 0;
    };
    std::vector<Part> parts(T);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            Part& P = parts[t];
            const char* a = cut[t];
            const char* b = cut[t + 1];
            P.r.reserve((size_t)(nnz_in / T + 16));
            P.c.reserve((size_t)(nnz_in / T + 16));
            P.v.reserve((size_t)(2 * (nnz_in / T + 16)));
            for (;;) {
                while (a < b && (*a == ' ' || *a == '\t' || *a == '\n' || *a == '\r')) ++a;
                if (a >= b) break;
                uint64_t r, c;
                double re, im;
                if (!parse_entry(a, b, r, c, re, im)) { P.err = 1; return; }
                if (r == 0 || c == 0) { P.err = 2; return; }
                P.r.push_back((int64_t)r - 1);
                P.c.push_back((int64_t)c - 1);
                P.v.push_back(re);
                P.v.push_back(im);
            }
        });
    for (auto& x : th) x.join();
    int64_t total = 0;
    for (const Part& P : parts) {
        if (P.err == 2) return cvk_fail(CVK_EINVAL, "matrix market: indices are 1-based");
        if (P.err) return cvk_fail(CVK_EINVAL, "matrix market: truncated entry list");
        total += (int64_t)P.r.size();
    }
    // the reference reads exactly nnz entries and ignores anything after them
    if (total < nnz_in) return cvk_fail(CVK_EINVAL, "matrix market: truncated entry list");
    // range check (csr_from_triplets, numkit.cpp:44-48) over the first nnz entries
    std::vector<int64_t> base(T + 1, 0);
    for (int t = 0; t < T; ++t) base[t + 1] = base[t] + (int64_t)parts[t].r.size();
    for (int t = 0; t < T; ++t)
        for (size_t k = 0; k < parts[t].r.size() && base[t] + (int64_t)k < nnz_in; ++k)
            if (parts[t].r[k] >= nrows || parts[t].c[k] >= ncols)
                return cvk_fail(CVK_EINVAL, "csr_from_triplets: index out of range at (" +
                                                std::to_string(parts[t].r[k]) + ", " + std::to_string(parts[t].c[k]) + ")");
    // counting sort by row, stable in input order
    std::vector<uint64_t> cnt((size_t)nrows + 1, 0);
    for (int t = 0; t < T; ++t)
        for (size_t k = 0; k < parts[t].r.size() && base[t] + (int64_t)k < nnz_in; ++k) cnt[(size_t)parts[t].r[k] + 1]++;
    for (int64_t i = 0; i < nrows; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
    std::vector<int64_t> col((size_t)nnz_in);
    std::vector<double> val((size_t)2 * nnz_in);
    {
        std::vector<uint64_t> pos(cnt.begin(), cnt.end() - 1);
        for (int t = 0; t < T; ++t) {
            const Part& P = parts[t];
            for (size_t k = 0; k < P.r.size() && base[t] + (int64_t)k < nnz_in; ++k) {
                const uint64_t d = pos[(size_t)P.r[k]]++;
                col[d] = P.c[k];
                val[2 * d] = P.v[2 * k];
                val[2 * d + 1] = P.v[2 * k + 1];
            }
        }
    }
    parts.clear();
    parts.shrink_to_fit();
    // per row: stable sort by column, sum duplicates in input order
    std::vector<uint64_t> ucnt((size_t)nrows + 1, 0);
    {
        std::vector<std::thread> th2;
        for (int t = 0; t < T; ++t)
            th2.emplace_back([&, t] {
                std::vector<int> idx;
                std::vector<int64_t> c2;
                std::vector<double> v2;
                for (int64_t i = nrows * t / T; i < nrows * (t + 1) / T; ++i) {
                    const uint64_t a = cnt[(size_t)i], b = cnt[(size_t)i + 1];
                    const int len = (int)(b - a);
                    idx.resize(len);
                    for (int k = 0; k < len; ++k) idx[k] = k;
                    std::stable_sort(idx.begin(), idx.end(),
                                     [&](int x, int y) { return col[a + x] < col[a + y]; });
                    c2.clear();
                    v2.clear();
                    for (int k = 0; k < len; ++k) {
                        const uint64_t q = a + idx[k];
                        if (!c2.empty() && c2.back() == col[q]) {
                            v2[v2.size() - 2] += val[2 * q];
                            v2[v2.size() - 1] += val[2 * q + 1];
                        } else {
                            c2.push_back(col[q]);
                            v2.push_back(val[2 * q]);
                            v2.push_back(val[2 * q + 1]);
                        }
                    }
                    for (size_t k = 0; k < c2.size(); ++k) {  // in place: the merged row is no longer
                        col[a + k] = c2[k];
                        val[2 * (a + k)] = v2[2 * k];
                        val[2 * (a + k) + 1] = v2[2 * k + 1];
                    }
                    ucnt[(size_t)i + 1] = c2.size();
                }
            });
        for (auto& x : th2) x.join();
    }
    for (int64_t i = 0; i < nrows; ++i) ucnt[(size_t)i + 1] += ucnt[(size_t)i];
    const int64_t nnz = (int64_t)ucnt[(size_t)nrows];
    uint64_t* rp = (uint64_t*)std::malloc(sizeof(uint64_t) * ((size_t)nrows + 1));
    uint64_t* ci = (uint64_t*)std::malloc(sizeof(uint64_t) * std::max<int64_t>(1, nnz));
    double* vv = (double*)std::malloc(sizeof(double) * 2 * std::max<int64_t>(1, nnz));
    if (!rp || !ci || !vv) {
        std::free(rp); std::free(ci); std::free(vv);
        return cvk_fail(CVK_ENOMEM, "cvk_mm_read: out of host memory");
    }
    std::memcpy(rp, ucnt.data(), sizeof(uint64_t) * ((size_t)nrows + 1));
    {
        std::vector<std::thread> th3;
        for (int t = 0; t < T; ++t)
            th3.emplace_back([&, t] {
                for (int64_t i = nrows * t / T; i < nrows * (t + 1) / T; ++i) {
                    const uint64_t a = cnt[(size_t)i], o = ucnt[(size_t)i], len = ucnt[(size_t)i + 1] - o;
                    for (uint64_t k = 0; k < len; ++k) {
                        ci[o + k] = (uint64_t)col[a + k];
                        vv[2 * (o + k)] = val[2 * (a + k)];
                        vv[2 * (o + k) + 1] = val[2 * (a + k) + 1];
                    }
                }
            });
        for (auto& x : th3) x.join();
    }
    out->nrows = nrows;
    out->ncols = ncols;
    out->nnz = nnz;
    out->row_offsets = rp;
    out->col_indices = ci;
    out->values = vv;
    return CVK_OK;
}

extern "C" void cvk_mm_free(cvk_mm_matrix* m) {
    if (!m) return;
    std::free(m->row_offsets);
    std::free(m->col_indices);
    std::free(m->values);
    std::memset(m, 0, sizeof(*m));
}

extern "C" int cvk_mm_write(const char* path, const cvk_mm_matrix* m, int nthreads) {
    if (!path || !m || (m->nrows > 0 && !m->row_offsets)) return cvk_fail(CVK_EINVAL, "cvk_mm_write: null argument");
    FILE* f = std::fopen(path, "wb");
    if (!f) return cvk_fail(CVK_EINVAL, std::string("cannot open ") + path + " for writing");
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate complex general\n%" PRId64 " %" PRId64 " %" PRId64 "\n",
                 m->nrows, m->ncols, m->nnz);
    // rows formatted in parallel blocks, written in order
    const int T = nthreads_for(nthreads);
    const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(m->nrows, (int64_t)T * 8));
    int rc = CVK_OK;
    for (int64_t b0 = 0; b0 < nb && rc == CVK_OK; b0 += T) {
        const int64_t b1 = std::min<int64_t>(nb, b0 + T);
        std::vector<std::string> buf((size_t)(b1 - b0));
        std::vector<std::thread> th;
        for (int64_t b = b0; b < b1; ++b)
            th.emplace_back([&, b] {
                std::string& o = buf[(size_t)(b - b0)];
                char tmp[160];
                for (int64_t i = m->nrows * b / nb; i < m->nrows * (b + 1) / nb; ++i)
                    for (uint64_t k = m->row_offsets[i]; k < m->row_offsets[i + 1]; ++k) {
                        const int len = std::snprintf(tmp, sizeof(tmp), "%" PRId64 " %" PRIu64 " %.17g %.17g\n", i + 1,
                                                      m->col_indices[k] + 1, m->values[2 * k], m->values[2 * k + 1]);
                        o.append(tmp, (size_t)len);
                    }
            });
        for (auto& x : th) x.join();
        for (const std::string& o : buf)
            if (std::fwrite(o.data(), 1, o.size(), f) != o.size()) { rc = CVK_EINVAL; break; }
    }
    if (std::fclose(f) != 0 || rc != CVK_OK) return cvk_fail(CVK_EINVAL, std::string("cannot write ") + path);
    return CVK_OK;
}
