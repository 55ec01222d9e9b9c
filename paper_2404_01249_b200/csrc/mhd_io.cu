// mhd_io.cu — MetaImage (.mhd + .raw) reader/writer of the reference's I/O
// layer (io.hpp, io.cpp:117-328) and a streaming device feed.
//
// Host-side format code follows io.cpp: "Key = value" header lines, NDims /
// DimSize / ElementType / ElementDataFile required, ElementSpacing / Offset /
// ElementNumberOfChannels optional, payload in a separate .raw next to the
// header; MET_FLOAT images and fields (channels interleaved), MET_SHORT
// labels.  Errors carry the reference's "path: byte N: ..." messages.
//
// The device feed (dfm_dev_load_image_mhd / dfm_dev_save_field_mhd) moves the
// fp32 payload between the file and HBM through two pinned chunk buffers, so
// the read of chunk k+1 overlaps the host->device copy of chunk k (and the
// device->host copy with the write on save); conversion to the context
// precision and the SoA <-> interleaved reshuffle run on the device.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/difform_gpu.h"
#include "dfm_kernels.cuh"

dfm_status dfm_internal_set_error(dfm_status code, const char* msg);  // engine.cu
// device-side helpers of engine.cu
dfm_status dfm_internal_ctx_info(dfm_ctx* ctx, int* precision, cudaStream_t* stream);
void* dfm_internal_ctx_buffer(dfm_ctx* ctx, const char* name, size_t bytes);
void dfm_internal_bump(dfm_ctx* ctx);

namespace {

struct IoError {
    int code;
    std::string msg;
};

[[noreturn]] void invalid(const std::string& m) { throw IoError{DFM_E_INVALID, m}; }
[[noreturn]] void runtime(const std::string& m) { throw IoError{DFM_E_NUMERICAL, m}; }

template <class F>
dfm_status io_guarded(F&& f) {
    try {
        f();
        return DFM_OK;
    } catch (const IoError& e) {
        return dfm_internal_set_error(static_cast<dfm_status>(e.code), e.msg.c_str());
    } catch (const std::exception& e) {
        return dfm_internal_set_error(DFM_E_CUDA, e.what());
    }
}

std::string fmt17(double v) {  // io.cpp:22-26
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

std::string trim(const std::string& s) {
    const size_t a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    const size_t b = s.find_last_not_of(" \t\r\n");
    return s.substr(a, b - a + 1);
}

std::string read_all(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) invalid(path + ": cannot open for reading");
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

void write_all(const std::string& path, const void* data, size_t n) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) invalid(path + ": cannot open for writing");
    out.write(static_cast<const char*>(data), static_cast<std::streamsize>(n));
    if (!out) runtime(path + ": write failed");
}

struct Line {
    std::string key, value;
    size_t offset = 0;
};

std::vector<Line> parse_lines(const std::string& text, const std::string& path) {
    std::vector<Line> out;
    size_t pos = 0;
    while (pos < text.size()) {
        const size_t eol = text.find('\n', pos);
        const size_t end = eol == std::string::npos ? text.size() : eol;
        const std::string line = trim(text.substr(pos, end - pos));
        if (!line.empty()) {
            const size_t eq = line.find('=');
            if (eq == std::string::npos)
                invalid(path + ": byte " + std::to_string(pos) + ": expected 'Key = value'");
            Line h;
            h.key = trim(line.substr(0, eq));
            h.value = trim(line.substr(eq + 1));
            h.offset = pos;
            if (h.key.empty()) invalid(path + ": byte " + std::to_string(pos) + ": empty key");
            out.push_back(h);
        }
        pos = eol == std::string::npos ? text.size() : eol + 1;
    }
    return out;
}

const Line* find(const std::vector<Line>& ls, const std::string& k) {
    for (const Line& h : ls)
        if (h.key == k) return &h;
    return nullptr;
}

const Line& require(const std::vector<Line>& ls, const std::string& k, const std::string& path) {
    const Line* h = find(ls, k);
    if (!h) invalid(path + ": byte 0: missing required key '" + k + "'");
    return *h;
}

std::vector<double> numbers(const Line& h, int expect, const std::string& path) {
    std::istringstream ss(h.value);
    std::vector<double> out;
    double v;
    while (ss >> v) out.push_back(v);
    std::string rest;
    if (ss.clear(), ss >> rest)
        invalid(path + ": byte " + std::to_string(h.offset) + ": non-numeric token in '" + h.key +
                "'");
    if (static_cast<int>(out.size()) != expect)
        invalid(path + ": byte " + std::to_string(h.offset) + ": '" + h.key + "' needs " +
                std::to_string(expect) + " values");
    return out;
}

std::string raw_path_for(const std::string& mhd) {
    std::filesystem::path p(mhd);
    p.replace_extension(".raw");
    return p.string();
}

void validate_meta(const dfm_grid& m, const std::string& prefix) {  // core.cpp:26-37
    std::string e;
    if (m.ndim != 2 && m.ndim != 3) e = "grid must have 2 or 3 axes";
    for (int a = 0; e.empty() && a < m.ndim; ++a) {
        if (m.dims[a] < 2) e = "grid dims must be >= 2 per axis";
        else if (!(m.spacing[a] > 0.0) || !std::isfinite(m.spacing[a])) e = "grid spacing must be > 0";
    }
    if (e.empty() && m.ndim == 2 && m.dims[2] != 1) e = "2D grid must have dims[2] == 1";
    if (!e.empty()) invalid(prefix + e);
}

// io.cpp:152-226
dfm_mhd_info read_header(const std::string& path) {
    const std::vector<Line> lines = parse_lines(read_all(path), path);
    dfm_mhd_info info{};
    const Line& nd = require(lines, "NDims", path);
    const double ndv = numbers(nd, 1, path)[0];
    if (ndv != 2.0 && ndv != 3.0)
        invalid(path + ": byte " + std::to_string(nd.offset) + ": NDims must be 2 or 3");
    dfm_grid& m = info.grid;
    m.ndim = static_cast<int32_t>(ndv);
    for (int a = 0; a < 3; ++a) {
        m.dims[a] = 1;
        m.spacing[a] = 1.0;
        m.origin[a] = 0.0;
    }
    const Line& ds = require(lines, "DimSize", path);
    const std::vector<double> dims = numbers(ds, m.ndim, path);
    for (int a = 0; a < m.ndim; ++a) {
        if (dims[a] < 1 || dims[a] != std::floor(dims[a]))
            invalid(path + ": byte " + std::to_string(ds.offset) +
                    ": DimSize entries must be positive integers");
        m.dims[a] = static_cast<int64_t>(dims[a]);
    }
    if (const Line* sp = find(lines, "ElementSpacing")) {
        const std::vector<double> v = numbers(*sp, m.ndim, path);
        for (int a = 0; a < m.ndim; ++a) m.spacing[a] = v[a];
    }
    if (const Line* of = find(lines, "Offset")) {
        const std::vector<double> v = numbers(*of, m.ndim, path);
        for (int a = 0; a < m.ndim; ++a) m.origin[a] = v[a];
    }
    validate_meta(m, path + ": byte 0: ");
    const Line& et = require(lines, "ElementType", path);
    info.element_type = et.value == "MET_FLOAT" ? DFM_MET_FLOAT
                        : et.value == "MET_SHORT" ? DFM_MET_SHORT
                                                  : DFM_MET_OTHER;
    std::strncpy(info.element_type_name, et.value.c_str(), sizeof(info.element_type_name) - 1);
    info.channels = 1;
    if (const Line* ch = find(lines, "ElementNumberOfChannels")) {
        const double c = numbers(*ch, 1, path)[0];
        if (c < 1 || c != std::floor(c))
            invalid(path + ": byte " + std::to_string(ch->offset) +
                    ": ElementNumberOfChannels must be a positive integer");
        info.channels = static_cast<int32_t>(c);
    }
    const Line& df = require(lines, "ElementDataFile", path);
    if (df.value.empty() || df.value == "LOCAL")
        invalid(path + ": byte " + std::to_string(df.offset) +
                ": embedded payloads are not supported");
    std::filesystem::path rp(df.value);
    if (rp.is_relative()) rp = std::filesystem::path(path).parent_path() / rp;
    const std::string r = rp.string();
    if (r.size() >= sizeof(info.raw_path)) invalid(path + ": byte 0: data file path too long");
    std::strncpy(info.raw_path, r.c_str(), sizeof(info.raw_path) - 1);
    return info;
}

// io.cpp:117-140
void write_header(const std::string& path, const dfm_grid& m, const char* type, int channels) {
    std::ostringstream h;
    h << "ObjectType = Image\n";
    h << "NDims = " << m.ndim << "\n";
    h << "DimSize =";
    for (int a = 0; a < m.ndim; ++a) h << " " << m.dims[a];
    h << "\nElementSpacing =";
    for (int a = 0; a < m.ndim; ++a) h << " " << fmt17(m.spacing[a]);
    h << "\nOffset =";
    for (int a = 0; a < m.ndim; ++a) h << " " << fmt17(m.origin[a]);
    h << "\nElementType = " << type << "\n";
    if (channels > 1) h << "ElementNumberOfChannels = " << channels << "\n";
    h << "ElementDataFile = " << std::filesystem::path(raw_path_for(path)).filename().string()
      << "\n";
    const std::string s = h.str();
    write_all(path, s.data(), s.size());
}

int64_t voxels(const dfm_grid& g) { return g.dims[0] * g.dims[1] * g.dims[2]; }

// typed header + exact payload size (io.cpp:218-226, 245-328)
dfm_mhd_info open_typed(const std::string& path, int type, int channels_expect, size_t esz,
                        const char* what) {
    dfm_mhd_info info = read_header(path);
    if (info.element_type != type)
        invalid(path + ": byte 0: expected ElementType " +
                std::string(type == DFM_MET_FLOAT ? "MET_FLOAT" : "MET_SHORT") + ", got " +
                info.element_type_name);
    const int want = channels_expect > 0 ? channels_expect : info.grid.ndim;
    if (info.channels != want) {
        if (channels_expect > 0)
            invalid(path + ": byte 0: " + what + " cannot have " + std::to_string(info.channels) +
                    " channels");
        invalid(path + ": byte 0: field needs " + std::to_string(want) + " channels, got " +
                std::to_string(info.channels));
    }
    std::ifstream in(info.raw_path, std::ios::binary | std::ios::ate);
    if (!in) invalid(std::string(info.raw_path) + ": cannot open for reading");
    const size_t bytes = static_cast<size_t>(in.tellg());
    const size_t expect = static_cast<size_t>(voxels(info.grid)) * want * esz;
    if (bytes != expect)
        invalid(std::string(info.raw_path) + ": byte " + std::to_string(bytes) + ": payload is " +
                std::to_string(bytes) + " bytes, expected " + std::to_string(expect));
    return info;
}

template <class T>
std::vector<T> read_payload(const dfm_mhd_info& info, size_t count) {
    std::vector<T> buf(count);
    std::ifstream in(info.raw_path, std::ios::binary);
    in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(count * sizeof(T)));
    if (!in) invalid(std::string(info.raw_path) + ": short read");
    return buf;
}

constexpr size_t kChunk = size_t(16) << 20;  // bytes per pinned staging chunk

}  // namespace

extern "C" {

dfm_status dfm_mhd_read_header(const char* path, dfm_mhd_info* out) {
    return io_guarded([&] { *out = read_header(path); });
}

dfm_status dfm_mhd_write_image(const char* path, const dfm_grid* g, const double* img) {
    return io_guarded([&] {
        validate_meta(*g, "");
        write_header(path, *g, "MET_FLOAT", 1);
        const int64_t n = voxels(*g);
        std::vector<float> buf(n);
        for (int64_t i = 0; i < n; ++i) buf[i] = static_cast<float>(img[i]);
        write_all(raw_path_for(path), buf.data(), buf.size() * sizeof(float));
    });
}

dfm_status dfm_mhd_read_image(const char* path, dfm_grid* g, double* out, int64_t capacity) {
    return io_guarded([&] {
        const dfm_mhd_info info = open_typed(path, DFM_MET_FLOAT, 1, 4, "scalar image");
        const int64_t n = voxels(info.grid);
        *g = info.grid;
        if (!out) return;  // size query
        if (capacity < n) invalid(std::string(path) + ": output buffer too small");
        const std::vector<float> src = read_payload<float>(info, n);
        for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(src[i]);
    });
}

dfm_status dfm_mhd_write_labels(const char* path, const dfm_grid* g, const int32_t* labels) {
    return io_guarded([&] {
        validate_meta(*g, "");
        const int64_t n = voxels(*g);
        std::vector<int16_t> buf(n);
        for (int64_t i = 0; i < n; ++i) {
            const int32_t v = labels[i];
            if (v < -32768 || v > 32767)
                invalid(std::string(path) + ": label value " + std::to_string(v) +
                        " does not fit MET_SHORT");
            buf[i] = static_cast<int16_t>(v);
        }
        write_header(path, *g, "MET_SHORT", 1);
        write_all(raw_path_for(path), buf.data(), buf.size() * sizeof(int16_t));
    });
}

dfm_status dfm_mhd_read_labels(const char* path, dfm_grid* g, int32_t* out, int64_t capacity) {
    return io_guarded([&] {
        const dfm_mhd_info info = open_typed(path, DFM_MET_SHORT, 1, 2, "label image");
        const int64_t n = voxels(info.grid);
        *g = info.grid;
        if (!out) return;
        if (capacity < n) invalid(std::string(path) + ": output buffer too small");
        const std::vector<int16_t> src = read_payload<int16_t>(info, n);
        for (int64_t i = 0; i < n; ++i) out[i] = static_cast<int32_t>(src[i]);
    });
}

dfm_status dfm_mhd_write_field(const char* path, const dfm_grid* g, const double* field) {
    return io_guarded([&] {
        validate_meta(*g, "");
        write_header(path, *g, "MET_FLOAT", g->ndim);
        const int64_t n = voxels(*g) * g->ndim;
        std::vector<float> buf(n);
        for (int64_t i = 0; i < n; ++i) buf[i] = static_cast<float>(field[i]);
        write_all(raw_path_for(path), buf.data(), buf.size() * sizeof(float));
    });
}

dfm_status dfm_mhd_read_field(const char* path, dfm_grid* g, double* out, int64_t capacity) {
    return io_guarded([&] {
        const dfm_mhd_info info = open_typed(path, DFM_MET_FLOAT, 0, 4, "field");
        const int64_t n = voxels(info.grid) * info.grid.ndim;
        *g = info.grid;
        if (!out) return;
        if (capacity < n) invalid(std::string(path) + ": output buffer too small");
        const std::vector<float> src = read_payload<float>(info, n);
        for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(src[i]);
    });
}

// file -> pinned chunk (host thread) -> HBM fp32 staging (copy engine) ->
// context precision (device cast); two chunk buffers so the read of chunk
// k+1 overlaps the copy of chunk k
dfm_status dfm_dev_load_image_mhd(dfm_ctx* ctx, const char* path, dfm_grid* g, void* d_out) {
    return io_guarded([&] {
        const dfm_mhd_info info = open_typed(path, DFM_MET_FLOAT, 1, 4, "scalar image");
        *g = info.grid;
        if (!d_out) return;
        int prec = 0;
        cudaStream_t st = nullptr;
        if (dfm_internal_ctx_info(ctx, &prec, &st) != DFM_OK) invalid("ctx is NULL");
        const int64_t n = voxels(info.grid);
        const size_t bytes = static_cast<size_t>(n) * 4;
        float* dst = prec == DFM_PREC_F32
                         ? static_cast<float*>(d_out)
                         : static_cast<float*>(dfm_internal_ctx_buffer(ctx, "mhd_stage", bytes));
        char* pin = static_cast<char*>(dfm_internal_ctx_buffer(ctx, "@pinned:mhd", 2 * kChunk));
        cudaEvent_t ev[2];
        for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        std::ifstream in(info.raw_path, std::ios::binary);
        size_t off = 0;
        int k = 0;
        bool ok = true;
        while (off < bytes && ok) {
            const size_t len = std::min(kChunk, bytes - off);
            char* buf = pin + (k & 1) * kChunk;
            if (k >= 2) cudaEventSynchronize(ev[k & 1]);  // the copy that used this buffer
            in.read(buf, static_cast<std::streamsize>(len));
            ok = static_cast<bool>(in);
            if (!ok) break;
            cudaMemcpyAsync(reinterpret_cast<char*>(dst) + off, buf, len, cudaMemcpyHostToDevice, st);
            cudaEventRecord(ev[k & 1], st);
            off += len;
            ++k;
        }
        if (prec == DFM_PREC_F64 && ok) {
            dfm::Launch L{st, nullptr, 0};
            dfm::launch_cast<double, float>(L, dst, static_cast<double*>(d_out), n);
            dfm_internal_bump(ctx);
        }
        const cudaError_t e = cudaStreamSynchronize(st);
        for (auto& q : ev) cudaEventDestroy(q);
        if (!ok) invalid(std::string(info.raw_path) + ": short read");
        if (e != cudaSuccess) throw IoError{DFM_E_CUDA, cudaGetErrorString(e)};
    });
}

// HBM SoA field (context precision) -> interleaved fp32 on the device ->
// pinned chunks -> file, the write of chunk k overlapping the copy of k+1
dfm_status dfm_dev_save_field_mhd(dfm_ctx* ctx, const char* path, const dfm_grid* g,
                                  const void* d_field_soa) {
    return io_guarded([&] {
        validate_meta(*g, "");
        int prec = 0;
        cudaStream_t st = nullptr;
        if (dfm_internal_ctx_info(ctx, &prec, &st) != DFM_OK) invalid("ctx is NULL");
        const int64_t n = voxels(*g);
        const int nd = g->ndim;
        const size_t bytes = static_cast<size_t>(n) * nd * 4;
        float* aos = static_cast<float*>(dfm_internal_ctx_buffer(ctx, "mhd_stage", bytes));
        dfm::Launch L{st, nullptr, 0};
        if (prec == DFM_PREC_F32) {
            const float* u = static_cast<const float*>(d_field_soa);
            dfm::launch_soa_to_aos<float, float>(L, dfm::CPlanes3<float>{{u, u + n, u + 2 * n}},
                                                 aos, n, nd);
        } else {
            const double* u = static_cast<const double*>(d_field_soa);
            dfm::launch_soa_to_aos<double, float>(
                L, dfm::CPlanes3<double>{{u, u + n, u + 2 * n}}, aos, n, nd);
        }
        dfm_internal_bump(ctx);
        write_header(path, *g, "MET_FLOAT", nd);
        const std::string raw = raw_path_for(path);
        std::ofstream out(raw, std::ios::binary | std::ios::trunc);
        if (!out) invalid(raw + ": cannot open for writing");
        char* pin = static_cast<char*>(dfm_internal_ctx_buffer(ctx, "@pinned:mhd", 2 * kChunk));
        cudaEvent_t ev[2];
        for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        size_t nchunk = (bytes + kChunk - 1) / kChunk;
        auto issue = [&](size_t c) {
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            cudaMemcpyAsync(pin + (c & 1) * kChunk, reinterpret_cast<char*>(aos) + off, len,
                            cudaMemcpyDeviceToHost, st);
            cudaEventRecord(ev[c & 1], st);
        };
        if (nchunk > 0) issue(0);
        for (size_t c = 0; c < nchunk; ++c) {
            if (c + 1 < nchunk) issue(c + 1);  // next copy overlaps this write
            cudaEventSynchronize(ev[c & 1]);
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            out.write(pin + (c & 1) * kChunk, static_cast<std::streamsize>(len));
            if (c + 1 < nchunk) cudaEventSynchronize(ev[(c + 1) & 1]);
        }
        const cudaError_t e = cudaStreamSynchronize(st);
        for (auto& q : ev) cudaEventDestroy(q);
        if (!out) runtime(raw + ": write failed");
        if (e != cudaSuccess) throw IoError{DFM_E_CUDA, cudaGetErrorString(e)};
    });
}

}  // extern "C"
