// hysco_io.cu -- NIfTI-1 volume I/O and the PE-last permutation (SURVEY §8(f)
// NEXT-4; include/hysco_io.h).  Host code (zlib) plus one GPU kernel: a
// batched 2-D transpose through shared memory that moves the PE axis of the
// file order [nz][ny][nx] to the last (contiguous) position and back.
#include "hysco_io.h"

#include <cuda_runtime.h>
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <thread>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

hysco_status io_err(hysco_status s, const std::string& m) {
    g_err = m;
    return s;
}

// NIfTI-1 header field offsets (348-byte header)
enum : int {
    OFF_SIZEOF_HDR = 0, OFF_DIM = 40, OFF_DATATYPE = 70, OFF_BITPIX = 72, OFF_PIXDIM = 76, OFF_VOX_OFFSET = 108,
    OFF_SCL_SLOPE = 112, OFF_SCL_INTER = 116, OFF_XYZT_UNITS = 123, OFF_QFORM_CODE = 252, OFF_SFORM_CODE = 254,
    OFF_QUATERN_B = 256, OFF_QOFFSET_X = 268, OFF_SROW_X = 280, OFF_MAGIC = 344, HDR_SIZE = 348
};

template <typename V>
V rd(const unsigned char* h, int off) {
    V v;
    memcpy(&v, h + off, sizeof(V));
    return v;
}
template <typename V>
void wr(unsigned char* h, int off, V v) {
    memcpy(h + off, &v, sizeof(V));
}

int type_bytes(int dt) {
    switch (dt) {
        case 2: case 256: return 1;
        case 4: case 512: return 2;
        case 8: case 16: return 4;
        case 64: return 8;
        default: return 0;
    }
}

struct GzFile {
    gzFile f = nullptr;
    ~GzFile() {
        if (f) gzclose(f);
    }
};

hysco_status parse_header(const unsigned char* h, hysco_nifti_info* info, double* vox_offset) {
    const int32_t sz = rd<int32_t>(h, OFF_SIZEOF_HDR);
    if (sz != HDR_SIZE) {
        int32_t sw = (int32_t)__builtin_bswap32((uint32_t)sz);
        if (sw == HDR_SIZE) return io_err(HYSCO_ERR_ARG, "big-endian NIfTI files are not supported");
        return io_err(HYSCO_ERR_ARG, "not a NIfTI-1 file (sizeof_hdr != 348)");
    }
    if (memcmp(h + OFF_MAGIC, "n+1\0", 4) != 0)
        return io_err(HYSCO_ERR_ARG, "not a single-file NIfTI-1 (magic != \"n+1\")");
    const int16_t* dim = reinterpret_cast<const int16_t*>(h + OFF_DIM);
    int16_t d[8];
    memcpy(d, dim, sizeof d);
    if (!(d[0] == 3 || (d[0] == 4 && d[4] == 1)))
        return io_err(HYSCO_ERR_ARG, "only 3-D volumes (or 4-D with a singleton 4th dimension) are supported");
    for (int k = 1; k <= 3; k++)
        if (d[k] < 1) return io_err(HYSCO_ERR_ARG, "non-positive dimension");
    const int dt = rd<int16_t>(h, OFF_DATATYPE);
    if (!type_bytes(dt)) return io_err(HYSCO_ERR_ARG, "unsupported NIfTI datatype " + std::to_string(dt));
    float pd[8];
    memcpy(pd, h + OFF_PIXDIM, sizeof pd);
    hysco_nifti_info o;
    memset(&o, 0, sizeof o);
    for (int k = 0; k < 3; k++) {
        o.dim[k] = d[k + 1];
        o.pixdim[k] = pd[k + 1];
    }
    o.datatype = dt;
    o.scl_slope = rd<float>(h, OFF_SCL_SLOPE);
    o.scl_inter = rd<float>(h, OFF_SCL_INTER);
    o.qform_code = rd<int16_t>(h, OFF_QFORM_CODE);
    o.sform_code = rd<int16_t>(h, OFF_SFORM_CODE);
    o.qfac = pd[0] < 0 ? -1.0 : 1.0;
    for (int k = 0; k < 3; k++) {
        o.quatern[k] = rd<float>(h, OFF_QUATERN_B + 4 * k);
        o.qoffset[k] = rd<float>(h, OFF_QOFFSET_X + 4 * k);
    }
    for (int k = 0; k < 12; k++) o.srow[k] = rd<float>(h, OFF_SROW_X + 4 * k);
    if (info) *info = o;
    if (vox_offset) *vox_offset = rd<float>(h, OFF_VOX_OFFSET);
    return HYSCO_OK;
}

hysco_status open_read(const char* path, GzFile& g, unsigned char* hdr) {
    if (!path) return io_err(HYSCO_ERR_ARG, "path is NULL");
    g.f = gzopen(path, "rb");                 // zlib reads plain and gzip files alike
    if (!g.f) return io_err(HYSCO_ERR_ARG, std::string("cannot open ") + path);
    if (gzread(g.f, hdr, HDR_SIZE) != HDR_SIZE) return io_err(HYSCO_ERR_ARG, "truncated NIfTI header");
    return HYSCO_OK;
}

template <typename T>
hysco_status convert(const unsigned char* raw, int dt, size_t n, double slope, double inter, T* out) {
    const bool scale = slope != 0.0 && !(slope == 1.0 && inter == 0.0);
    for (size_t i = 0; i < n; i++) {
        double v;
        switch (dt) {
            case 2: v = raw[i]; break;
            case 256: v = (double)reinterpret_cast<const int8_t*>(raw)[i]; break;
            case 4: v = (double)reinterpret_cast<const int16_t*>(raw)[i]; break;
            case 512: v = (double)reinterpret_cast<const uint16_t*>(raw)[i]; break;
            case 8: v = (double)reinterpret_cast<const int32_t*>(raw)[i]; break;
            case 16: v = (double)reinterpret_cast<const float*>(raw)[i]; break;
            default: v = reinterpret_cast<const double*>(raw)[i]; break;
        }
        if (scale) v = v * slope + inter;
        if (!std::isfinite(v)) return io_err(HYSCO_ERR_ARG, "non-finite voxel value");
        out[i] = (T)v;
    }
    return HYSCO_OK;
}

template <typename T>
bool all_finite(const T* p, size_t n) {
    for (size_t i = 0; i < n; i++)
        if (!std::isfinite((double)p[i])) return false;
    return true;
}

// ---- GPU permutation ------------------------------------------------------
// out[b*sBo + c*sCo + r] = in[b*sBi + r*sRi + c] for r < R, c < C, b < NB,
// per volume (volume stride V in both).  32 x 32 tiles: reads coalesced along
// c, writes coalesced along r; the +1 padding avoids bank conflicts.
constexpr int PT = 32, PR = 8;

template <typename E>
__global__ void __launch_bounds__(PT * PR) permute_kernel(const E* __restrict__ in, E* __restrict__ out, long long R,
                                                          long long C, long long NB, long long sBi, long long sRi,
                                                          long long sBo, long long sCo, long long V) {
    __shared__ E tile[PT][PT + 1];
    const long long b = blockIdx.z % NB, vol = blockIdx.z / NB;
    const long long r0 = (long long)blockIdx.y * PT, c0 = (long long)blockIdx.x * PT;
    const E* src = in + vol * V + b * sBi;
    E* dst = out + vol * V + b * sBo;
    for (int y = threadIdx.y; y < PT; y += PR) {
        const long long r = r0 + y, c = c0 + threadIdx.x;
        if (r < R && c < C) tile[y][threadIdx.x] = src[r * sRi + c];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < PT; y += PR) {
        const long long c = c0 + y, r = r0 + threadIdx.x;
        if (r < R && c < C) dst[c * sCo + r] = tile[threadIdx.x][y];
    }
}

}  // namespace

extern "C" {

const char* hysco_io_last_error(void) { return g_err.c_str(); }

hysco_status hysco_nifti_info_read(const char* path, hysco_nifti_info* info) {
    GzFile g;
    unsigned char hdr[HDR_SIZE];
    if (hysco_status s = open_read(path, g, hdr)) return s;
    return parse_header(hdr, info, nullptr);
}

hysco_status hysco_nifti_read(const char* path, hysco_dtype dtype, void* host_out, int64_t n_elems,
                              hysco_nifti_info* info) {
    if (!host_out || (dtype != HYSCO_F32 && dtype != HYSCO_F64)) return io_err(HYSCO_ERR_ARG, "bad output / dtype");
    GzFile g;
    unsigned char hdr[HDR_SIZE];
    if (hysco_status s = open_read(path, g, hdr)) return s;
    hysco_nifti_info o;
    double vox = 0;
    if (hysco_status s = parse_header(hdr, &o, &vox)) return s;
    const size_t n = (size_t)o.dim[0] * o.dim[1] * o.dim[2];
    if ((int64_t)n != n_elems) return io_err(HYSCO_ERR_SHAPE, "n_elems does not match the file's dimensions");
    if (!(vox >= HDR_SIZE)) vox = 352;        // vox_offset 0 in a single file: data follows the extension flag
    const long skip = (long)vox - HDR_SIZE;
    std::vector<unsigned char> tmp((size_t)skip);
    if (skip > 0 && gzread(g.f, tmp.data(), (unsigned)skip) != (int)skip)
        return io_err(HYSCO_ERR_ARG, "truncated NIfTI file (before vox_offset)");
    const size_t nb = n * (size_t)type_bytes(o.datatype);
    std::vector<unsigned char> raw(nb);
    size_t got = 0;
    while (got < nb) {                         // gzread takes unsigned counts: read in chunks
        const unsigned chunk = (unsigned)std::min<size_t>(nb - got, (size_t)1 << 30);
        const int r = gzread(g.f, raw.data() + got, chunk);
        if (r <= 0) return io_err(HYSCO_ERR_ARG, "truncated NIfTI file (voxel data)");
        got += (size_t)r;
    }
    hysco_status s = dtype == HYSCO_F64
                         ? convert<double>(raw.data(), o.datatype, n, o.scl_slope, o.scl_inter, (double*)host_out)
                         : convert<float>(raw.data(), o.datatype, n, o.scl_slope, o.scl_inter, (float*)host_out);
    if (s) return s;
    if (info) *info = o;
    return HYSCO_OK;
}

hysco_status hysco_nifti_write(const char* path, hysco_dtype dtype, const void* host_data,
                               const hysco_nifti_info* info) {
    if (!path || !host_data || !info || (dtype != HYSCO_F32 && dtype != HYSCO_F64))
        return io_err(HYSCO_ERR_ARG, "bad arguments");
    for (int k = 0; k < 3; k++)
        if (info->dim[k] < 1 || info->dim[k] > 32767 || !(info->pixdim[k] > 0))
            return io_err(HYSCO_ERR_ARG, "dims must be in [1, 32767] and voxel sizes > 0");
    const size_t n = (size_t)info->dim[0] * info->dim[1] * info->dim[2];
    const bool f64 = dtype == HYSCO_F64;
    if (!(f64 ? all_finite((const double*)host_data, n) : all_finite((const float*)host_data, n)))
        return io_err(HYSCO_ERR_ARG, "non-finite voxel value");
    unsigned char h[352];
    memset(h, 0, sizeof h);
    wr<int32_t>(h, OFF_SIZEOF_HDR, HDR_SIZE);
    int16_t d[8] = {3, (int16_t)info->dim[0], (int16_t)info->dim[1], (int16_t)info->dim[2], 1, 1, 1, 1};
    memcpy(h + OFF_DIM, d, sizeof d);
    wr<int16_t>(h, OFF_DATATYPE, f64 ? 64 : 16);
    wr<int16_t>(h, OFF_BITPIX, f64 ? 64 : 32);
    float pd[8] = {(float)(info->qfac < 0 ? -1.0 : 1.0), (float)info->pixdim[0], (float)info->pixdim[1],
                   (float)info->pixdim[2], 0, 0, 0, 0};
    memcpy(h + OFF_PIXDIM, pd, sizeof pd);
    wr<float>(h, OFF_VOX_OFFSET, 352.0f);
    wr<float>(h, OFF_SCL_SLOPE, 1.0f);
    wr<float>(h, OFF_SCL_INTER, 0.0f);
    h[OFF_XYZT_UNITS] = 2;                     // NIFTI_UNITS_MM
    wr<int16_t>(h, OFF_QFORM_CODE, (int16_t)info->qform_code);
    wr<int16_t>(h, OFF_SFORM_CODE, (int16_t)info->sform_code);
    for (int k = 0; k < 3; k++) {
        wr<float>(h, OFF_QUATERN_B + 4 * k, (float)info->quatern[k]);
        wr<float>(h, OFF_QOFFSET_X + 4 * k, (float)info->qoffset[k]);
    }
    for (int k = 0; k < 12; k++) wr<float>(h, OFF_SROW_X + 4 * k, (float)info->srow[k]);
    memcpy(h + OFF_MAGIC, "n+1\0", 4);
    const std::string p(path);
    const bool gz = p.size() >= 3 && p.compare(p.size() - 3, 3, ".gz") == 0;
    const size_t nb = n * (f64 ? 8 : 4);
    const unsigned char* src = (const unsigned char*)host_data;
    if (gz) {
        // Independent gzip members of <= 1 MiB compressed by parallel threads at
        // level 1 (nibabel's default), concatenated: RFC 1952 allows several
        // members and zlib's gzread (and gunzip) reads them as one stream.
        std::vector<unsigned char> all(sizeof h + nb);
        memcpy(all.data(), h, sizeof h);
        memcpy(all.data() + sizeof h, src, nb);
        const size_t CH = (size_t)1 << 20, nch = (all.size() + CH - 1) / CH;
        std::vector<std::vector<unsigned char>> out(nch);
        std::vector<int> ok(nch, 0);
        const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 16u));
        std::atomic<size_t> next{0};
        auto work = [&]() {
            for (size_t c; (c = next.fetch_add(1)) < nch;) {
                const size_t off = c * CH, len = std::min(CH, all.size() - off);
                z_stream zs;
                memset(&zs, 0, sizeof zs);
                if (deflateInit2(&zs, 1, Z_DEFLATED, 15 + 16, 8, Z_DEFAULT_STRATEGY) != Z_OK) continue;
                out[c].resize(deflateBound(&zs, (uLong)len) + 64);
                zs.next_in = all.data() + off;
                zs.avail_in = (uInt)len;
                zs.next_out = out[c].data();
                zs.avail_out = (uInt)out[c].size();
                const int r = deflate(&zs, Z_FINISH);
                out[c].resize(out[c].size() - zs.avail_out);
                deflateEnd(&zs);
                ok[c] = r == Z_STREAM_END;
            }
        };
        std::vector<std::thread> th;
        for (unsigned t = 1; t < nt; t++) th.emplace_back(work);
        work();
        for (auto& t : th) t.join();
        for (size_t c = 0; c < nch; c++)
            if (!ok[c]) return io_err(HYSCO_ERR_ARG, "gzip compression failed");
        FILE* f = fopen(path, "wb");
        if (!f) return io_err(HYSCO_ERR_ARG, std::string("cannot create ") + path);
        bool good = true;
        for (size_t c = 0; c < nch && good; c++) good = fwrite(out[c].data(), 1, out[c].size(), f) == out[c].size();
        good = (fclose(f) == 0) && good;
        return good ? HYSCO_OK : io_err(HYSCO_ERR_ARG, "write failed");
    }
    FILE* f = fopen(path, "wb");
    if (!f) return io_err(HYSCO_ERR_ARG, std::string("cannot create ") + path);
    bool good = fwrite(h, 1, sizeof h, f) == sizeof h && fwrite(src, 1, nb, f) == nb;
    good = (fclose(f) == 0) && good;
    return good ? HYSCO_OK : io_err(HYSCO_ERR_ARG, "write failed");
}

hysco_status hysco_pe_shape(const int64_t dims[3], const double pixdim[3], int32_t pe_axis, int64_t n_out[3],
                            double h_out[3]) {
    if (!dims || !n_out || pe_axis < 1 || pe_axis > 3) return io_err(HYSCO_ERR_ARG, "pe_axis must be 1, 2 or 3");
    static const int order[3][3] = {{2, 1, 0}, {2, 0, 1}, {1, 0, 2}};   // NIfTI axes (0 = x) of (n1, n2, n3)
    for (int k = 0; k < 3; k++) {
        n_out[k] = dims[order[pe_axis - 1][k]];
        if (h_out && pixdim) h_out[k] = pixdim[order[pe_axis - 1][k]];
    }
    return HYSCO_OK;
}

hysco_status hysco_permute_pe(const void* d_in, void* d_out, const int64_t dims[3], int32_t pe_axis, int32_t inverse,
                              hysco_dtype dtype, int64_t batch, void* cuda_stream) {
    if (!d_in || !d_out || !dims || pe_axis < 1 || pe_axis > 3 || batch < 1 ||
        (dtype != HYSCO_F32 && dtype != HYSCO_F64))
        return io_err(HYSCO_ERR_ARG, "bad arguments");
    const long long nx = dims[0], ny = dims[1], nz = dims[2];
    if (nx < 1 || ny < 1 || nz < 1) return io_err(HYSCO_ERR_SHAPE, "non-positive dimension");
    const long long V = nx * ny * nz;
    const size_t esz = dtype == HYSCO_F64 ? 8 : 4;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if (pe_axis == 1) {
        const cudaError_t e = cudaMemcpyAsync(d_out, d_in, (size_t)(V * batch) * esz, cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? HYSCO_OK : io_err(HYSCO_ERR_CUDA, cudaGetErrorString(e));
    }
    // (R, C, NB, sBi, sRi, sBo, sCo) of the batched transpose (derivation in DESIGN.md §7)
    long long R, C, NB, sBi, sRi, sBo, sCo;
    if (pe_axis == 2 && !inverse) {            // [nz][ny][nx] -> [nz][nx][ny]
        R = ny; C = nx; NB = nz; sBi = ny * nx; sRi = nx; sBo = nx * ny; sCo = ny;
    } else if (pe_axis == 2) {                 // [nz][nx][ny] -> [nz][ny][nx]
        R = nx; C = ny; NB = nz; sBi = nx * ny; sRi = ny; sBo = ny * nx; sCo = nx;
    } else if (!inverse) {                     // [nz][ny][nx] -> [ny][nx][nz]
        R = nz; C = nx; NB = ny; sBi = nx; sRi = ny * nx; sBo = nx * nz; sCo = nz;
    } else {                                   // [ny][nx][nz] -> [nz][ny][nx]
        R = nx; C = nz; NB = ny; sBi = nx * nz; sRi = nz; sBo = nx; sCo = ny * nx;
    }
    if (NB * batch > 2147483647LL || (R + PT - 1) / PT > 65535) return io_err(HYSCO_ERR_SHAPE, "volume too large");
    const dim3 grid((unsigned)((C + PT - 1) / PT), (unsigned)((R + PT - 1) / PT), (unsigned)(NB * batch));
    if (NB * batch > 65535) return io_err(HYSCO_ERR_SHAPE, "too many planes for one launch");
    if (esz == 8)
        permute_kernel<double><<<grid, dim3(PT, PR), 0, st>>>((const double*)d_in, (double*)d_out, R, C, NB, sBi,
                                                              sRi, sBo, sCo, V);
    else
        permute_kernel<float><<<grid, dim3(PT, PR), 0, st>>>((const float*)d_in, (float*)d_out, R, C, NB, sBi, sRi,
                                                             sBo, sCo, V);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HYSCO_OK : io_err(HYSCO_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
