// formats.cpp — the reference's interchange formats behind the C ABI, so the GPU path reads
// and writes the same files as the reference CLI pipeline:
//
//   * VSTN tensors       — tensor_io.hpp:14-88 (+ binio.hpp little-endian primitives)
//   * VSCK checkpoints   — indexer.hpp:450-499 (one indexer per KV head)
//   * "V:"/"S:" indices  — sparsity.hpp:187-245
//
// Host-only code; no device work happens here (the Python mirror moves the arrays to HBM).
// Error codes follow the reference's exception types: std::runtime_error → VSP_ERUNTIME,
// std::invalid_argument → VSP_EINVAL, with the reference's message text verbatim.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vsp_gpu.h"
#include "vsp_error.h"

namespace {

using vsp_detail::set_err;

// Little-endian byte order regardless of host (binio.hpp:12-50).
void put_u32(std::string& buf, uint32_t x) {
    for (int i = 0; i < 4; ++i) buf.push_back(static_cast<char>((x >> (8 * i)) & 0xff));
}
void put_u64(std::string& buf, uint64_t x) {
    for (int i = 0; i < 8; ++i) buf.push_back(static_cast<char>((x >> (8 * i)) & 0xff));
}
void put_f64(std::string& buf, double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    put_u64(buf, u);
}

// A whole file in memory with a cursor; every short read reports the caller's message.
struct Reader {
    std::vector<unsigned char> bytes;
    size_t pos = 0;
    bool take(void* out, size_t nb) {
        if (bytes.size() - pos < nb) {
            pos = bytes.size();
            return false;
        }
        std::memcpy(out, bytes.data() + pos, nb);
        pos += nb;
        return true;
    }
    bool u32(uint32_t* x) {
        unsigned char b[4];
        if (!take(b, 4)) return false;
        *x = 0;
        for (int i = 0; i < 4; ++i) *x |= static_cast<uint32_t>(b[i]) << (8 * i);
        return true;
    }
    bool u64(uint64_t* x) {
        unsigned char b[8];
        if (!take(b, 8)) return false;
        *x = 0;
        for (int i = 0; i < 8; ++i) *x |= static_cast<uint64_t>(b[i]) << (8 * i);
        return true;
    }
    bool f64(double* x) {
        uint64_t u;
        if (!u64(&u)) return false;
        std::memcpy(x, &u, 8);
        return true;
    }
};

bool slurp(const char* path, Reader* r) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    unsigned char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) r->bytes.insert(r->bytes.end(), chunk, chunk + got);
    std::fclose(f);
    return true;
}

// Writes `buf` to `path`; the reference opens, streams, then checks the stream state once.
int spill(const char* path, const std::string& buf, const std::string& open_msg, const std::string& fail_msg) {
    FILE* f = std::fopen(path, "wb");
    if (!f) return set_err(VSP_ERUNTIME, open_msg);
    const size_t wrote = std::fwrite(buf.data(), 1, buf.size(), f);
    const int closed = std::fclose(f);
    if (wrote != buf.size() || closed != 0) return set_err(VSP_ERUNTIME, fail_msg);
    return VSP_OK;
}

// detail::read_tensor_header (tensor_io.hpp:26-42).
int read_vstn_header(Reader* r, const std::string& path, std::vector<uint64_t>* dims) {
    const std::string trunc = "truncated header in " + path;
    char magic[4];
    if (!r->take(magic, 4)) return set_err(VSP_ERUNTIME, trunc);
    if (std::memcmp(magic, "VSTN", 4) != 0) return set_err(VSP_ERUNTIME, "not a VSTN tensor: " + path);
    uint32_t version, ndim;
    if (!r->u32(&version)) return set_err(VSP_ERUNTIME, trunc);
    if (version != 1)
        return set_err(VSP_ERUNTIME, "unsupported VSTN version " + std::to_string(version) + " in " + path);
    if (!r->u32(&ndim)) return set_err(VSP_ERUNTIME, trunc);
    if (static_cast<uint64_t>(ndim) * 8 > r->bytes.size() - r->pos) return set_err(VSP_ERUNTIME, trunc);
    dims->assign(ndim, 0);
    for (uint64_t& d : *dims)
        if (!r->u64(&d)) return set_err(VSP_ERUNTIME, trunc);
    return VSP_OK;
}

int rank_error(size_t rank, int want, const std::string& path) {
    const char* what = want == 2 ? "rank-2 matrix" : "rank-1 vector";
    if (want != 1 && want != 2)
        return set_err(VSP_ERUNTIME, "tensor rank " + std::to_string(rank) + " where a rank-" +
                                         std::to_string(want) + " tensor was expected: " + path);
    return set_err(VSP_ERUNTIME, "tensor rank " + std::to_string(rank) + " where a " + what +
                                     " was expected: " + path);
}

// detail::parse_index_line (sparsity.hpp:208-232) over one line of text.
int parse_index_line(const std::string& line_in, const std::string& prefix, int64_t* out, int64_t cap,
                     int64_t* count) {
    std::string line = line_in;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.compare(0, prefix.size(), prefix) != 0)
        return set_err(VSP_ERUNTIME, "indices: expected '" + prefix + "' line, got '" + line + "'");
    // `rest >> long long` semantics: skip whitespace, optional sign, digits; stop at the first
    // token that is not a number (then eof() is false → "bad token").
    const char* p = line.c_str() + prefix.size();
    int64_t k = 0;
    for (;;) {
        while (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\v' || *p == '\f' || *p == '\r') ++p;
        if (*p == '\0') break;
        bool neg = false;
        if (*p == '+' || *p == '-') neg = (*p++ == '-');
        if (*p == '\0') break;  // a bare sign at end of line: the stream fails AT eof, no error
        if (*p < '0' || *p > '9') return set_err(VSP_ERUNTIME, "indices: bad token on '" + prefix + "' line");
        unsigned long long mag = 0;
        bool overflow = false;
        while (*p >= '0' && *p <= '9') {
            const unsigned d = static_cast<unsigned>(*p++ - '0');
            if (mag > (9223372036854775808ull - d) / 10) overflow = true;
            mag = mag * 10 + d;
        }
        if (overflow || (!neg && mag > 9223372036854775807ull)) {
            // out of range: the stream fails; only an overflow that ran to end of line leaves
            // eof() set (the reference then returns what it has read so far)
            if (*p == '\0') break;
            return set_err(VSP_ERUNTIME, "indices: bad token on '" + prefix + "' line");
        }
        if (neg && mag != 0) return set_err(VSP_ERUNTIME, "indices: negative index on '" + prefix + "' line");
        const int64_t v = static_cast<int64_t>(mag);
        if (k > 0 && v <= out[k - 1])
            return set_err(VSP_ERUNTIME, "indices: '" + prefix + "' line not strictly increasing");
        if (k >= cap) return set_err(VSP_EINVAL, "indices: capacity too small");
        out[k++] = v;
    }
    *count = k;
    return VSP_OK;
}

}  // namespace

extern "C" {

// ---- VSTN tensors (tensor_io.hpp) ------------------------------------------------------------

int vsp_tensor_header(const char* path, int* ndim, uint64_t* dims, int max_dims) {
    if (!path || !ndim) return set_err(VSP_EINVAL, "vsp_tensor_header: null argument");
    Reader r;
    if (!slurp(path, &r)) return set_err(VSP_ERUNTIME, std::string("cannot open tensor: ") + path);
    std::vector<uint64_t> d;
    if (int rc = read_vstn_header(&r, path, &d)) return rc;
    *ndim = static_cast<int>(d.size());
    for (int i = 0; i < max_dims && i < static_cast<int>(d.size()); ++i) dims[i] = d[i];
    return VSP_OK;
}

int vsp_read_tensor(const char* path, int rank, double* data, uint64_t count) {
    if (!path) return set_err(VSP_EINVAL, "vsp_read_tensor: null path");
    Reader r;
    if (!slurp(path, &r)) return set_err(VSP_ERUNTIME, std::string("cannot open tensor: ") + path);
    std::vector<uint64_t> d;
    if (int rc = read_vstn_header(&r, path, &d)) return rc;
    if (rank > 0 && d.size() != static_cast<size_t>(rank)) return rank_error(d.size(), rank, path);
    uint64_t want = 1;
    for (uint64_t x : d) want *= x;
    if (want != count)
        return set_err(VSP_EINVAL, "vsp_read_tensor: buffer holds " + std::to_string(count) + " values, file has " +
                                       std::to_string(want));
    const std::string trunc = std::string("truncated payload in ") + path;
    for (uint64_t i = 0; i < want; ++i)
        if (!r.f64(&data[i])) return set_err(VSP_ERUNTIME, trunc);
    return VSP_OK;
}

int vsp_write_tensor(const char* path, int ndim, const uint64_t* dims, const double* data) {
    if (!path || ndim < 0 || (ndim > 0 && !dims)) return set_err(VSP_EINVAL, "vsp_write_tensor: bad arguments");
    std::string buf("VSTN", 4);
    put_u32(buf, 1);
    put_u32(buf, static_cast<uint32_t>(ndim));
    uint64_t count = 1;
    for (int i = 0; i < ndim; ++i) {
        put_u64(buf, dims[i]);
        count *= dims[i];
    }
    if (count && !data) return set_err(VSP_EINVAL, "vsp_write_tensor: null data");
    buf.reserve(buf.size() + 8 * count);
    for (uint64_t i = 0; i < count; ++i) put_f64(buf, data[i]);
    return spill(path, buf, std::string("cannot open for writing: ") + path,
                 std::string("tensor write failed: ") + path);
}

// ---- VSCK checkpoints (indexer.hpp:450-499) ----------------------------------------------------

int vsp_checkpoint_header(const char* path, int* d, int* d_h) {
    if (!path || !d || !d_h) return set_err(VSP_EINVAL, "vsp_checkpoint_header: null argument");
    Reader r;
    if (!slurp(path, &r)) return set_err(VSP_ERUNTIME, std::string("cannot open checkpoint: ") + path);
    char magic[4];
    if (!r.take(magic, 4) || std::memcmp(magic, "VSCK", 4) != 0)
        return set_err(VSP_ERUNTIME, "not a VSCK checkpoint");
    uint32_t version, dd, dh;
    if (!r.u32(&version)) return set_err(VSP_ERUNTIME, "truncated checkpoint header");
    if (version != 1) return set_err(VSP_ERUNTIME, "unsupported VSCK version " + std::to_string(version));
    if (!r.u32(&dd) || !r.u32(&dh)) return set_err(VSP_ERUNTIME, "truncated checkpoint header");
    *d = static_cast<int>(dd);
    *d_h = static_cast<int>(dh);
    return VSP_OK;
}

int vsp_load_checkpoint(const char* path, int d, int d_h, double* w_u, double* b_u, double* w_v, double* b_v,
                        double* w_s, double* b_s) {
    int fd = 0, fdh = 0;
    if (int rc = vsp_checkpoint_header(path, &fd, &fdh)) return rc;
    if (fd != d || fdh != d_h)
        return set_err(VSP_EINVAL, "vsp_load_checkpoint: buffers sized for d=" + std::to_string(d) +
                                       ", d_h=" + std::to_string(d_h) + " but the checkpoint has d=" +
                                       std::to_string(fd) + ", d_h=" + std::to_string(fdh));
    Reader r;
    slurp(path, &r);
    r.pos = 16;
    bool ok = true;
    const size_t nw = static_cast<size_t>(2) * d * d_h;
    for (size_t i = 0; ok && i < nw; ++i) ok = r.f64(&w_u[i]);
    for (int i = 0; ok && i < d_h; ++i) ok = r.f64(&b_u[i]);
    for (int i = 0; ok && i < d_h; ++i) ok = r.f64(&w_v[i]);
    ok = ok && r.f64(b_v);
    for (int i = 0; ok && i < d_h; ++i) ok = r.f64(&w_s[i]);
    ok = ok && r.f64(b_s);
    if (!ok) return set_err(VSP_ERUNTIME, "truncated checkpoint payload");
    return VSP_OK;
}

int vsp_save_checkpoint(const char* path, int d, int d_h, const double* w_u, const double* b_u, const double* w_v,
                        double b_v, const double* w_s, double b_s) {
    if (!path) return set_err(VSP_EINVAL, "vsp_save_checkpoint: null path");
    if (d < 0 || d_h < 0 || (d_h > 0 && (!w_u || !b_u || !w_v || !w_s)))
        return set_err(VSP_EINVAL, "indexer params: inconsistent shapes");
    std::string buf("VSCK", 4);
    put_u32(buf, 1);
    put_u32(buf, static_cast<uint32_t>(d));
    put_u32(buf, static_cast<uint32_t>(d_h));
    const size_t nw = static_cast<size_t>(2) * d * d_h;
    buf.reserve(buf.size() + 8 * (nw + 3 * static_cast<size_t>(d_h) + 2));
    for (size_t i = 0; i < nw; ++i) put_f64(buf, w_u[i]);
    for (int i = 0; i < d_h; ++i) put_f64(buf, b_u[i]);
    for (int i = 0; i < d_h; ++i) put_f64(buf, w_v[i]);
    put_f64(buf, b_v);
    for (int i = 0; i < d_h; ++i) put_f64(buf, w_s[i]);
    put_f64(buf, b_s);
    return spill(path, buf, std::string("cannot open checkpoint for writing: ") + path,
                 std::string("checkpoint write failed: ") + path);
}

// ---- "V:" / "S:" index text (sparsity.hpp:187-245) ---------------------------------------------

int vsp_write_indices(const char* path, const int64_t* i_v, int64_t k_v, const int64_t* i_s, int64_t k_s) {
    if (!path || k_v < 0 || k_s < 0 || (k_v && !i_v) || (k_s && !i_s))
        return set_err(VSP_EINVAL, "vsp_write_indices: bad arguments");
    std::string buf = "V:";
    char num[32];
    for (int64_t t = 0; t < k_v; ++t) {
        std::snprintf(num, sizeof num, " %lld", static_cast<long long>(i_v[t]));
        buf += num;
    }
    buf += "\nS:";
    for (int64_t t = 0; t < k_s; ++t) {
        std::snprintf(num, sizeof num, " %lld", static_cast<long long>(i_s[t]));
        buf += num;
    }
    buf += '\n';
    FILE* f = std::fopen(path, "wb");
    if (!f) return set_err(VSP_ERUNTIME, std::string("cannot open for writing: ") + path);
    std::fwrite(buf.data(), 1, buf.size(), f);
    std::fclose(f);  // the reference does not check the stream after writing indices
    return VSP_OK;
}

int vsp_read_indices(const char* path, int64_t* i_v, int64_t* k_v, int64_t* i_s, int64_t* k_s, int64_t cap) {
    if (!path || !k_v || !k_s || cap < 0 || (cap && (!i_v || !i_s)))
        return set_err(VSP_EINVAL, "vsp_read_indices: bad arguments");
    Reader r;
    if (!slurp(path, &r)) return set_err(VSP_ERUNTIME, std::string("cannot open indices file: ") + path);
    // std::getline semantics: lines split on '\n'; a missing line is an error.
    std::string text(r.bytes.begin(), r.bytes.end());
    size_t at = 0;
    std::string lines[2];
    const char* prefixes[2] = {"V:", "S:"};
    int64_t* outs[2] = {i_v, i_s};
    int64_t* counts[2] = {k_v, k_s};
    for (int l = 0; l < 2; ++l) {
        if (at >= text.size()) return set_err(VSP_ERUNTIME, std::string("indices: missing '") + prefixes[l] + "' line");
        size_t nl = text.find('\n', at);
        if (nl == std::string::npos) nl = text.size();
        lines[l] = text.substr(at, nl - at);
        at = nl + 1;
        if (int rc = parse_index_line(lines[l], prefixes[l], outs[l], cap, counts[l])) return rc;
    }
    return VSP_OK;
}

}  // extern "C"
