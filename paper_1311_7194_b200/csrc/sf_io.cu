// sf_io.cu — DFRM depth-frame files (frame_io.cpp:28-79) to and from host or device buffers,
// and trajectory CSV files (frame_io.cpp:81-126). Host-side byte I/O; device frames are
// staged through one host copy.
#include <cstring>
#include <fstream>
#include <iomanip>
#include <sstream>
#include <string>
#include <vector>

#include "sf_internal.h"
#include "sf_linalg.cuh"

using namespace sf;

namespace {

template <typename T>
void put_raw(std::ofstream& o, const T& v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get_raw(std::ifstream& i) {
    T v{};
    i.read(reinterpret_cast<char*>(&v), sizeof(T));
    return v;
}

// is_rotation (pose.cpp:45-48): max |R^T R - I| and |det R - 1| within tol, in the Eigen
// evaluation order of the reference build (products summed left to right; 3x3 determinant by
// cofactors of the first column).
bool is_rotation_host(const m33& r, double tol) {
    const m33 rtr = mm(mt(r), r);
    double ortho = 0.0;
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k) {
            const double x = std::fabs(rtr.m[k * 3 + c] - (k == c ? 1.0 : 0.0));
            ortho = ortho < x ? x : ortho;
        }
    const double* m = r.m;
    const double det = m[0] * (m[4] * m[8] - m[7] * m[5]) - m[3] * (m[1] * m[8] - m[7] * m[2]) +
                       m[6] * (m[1] * m[5] - m[4] * m[2]);
    return ortho <= tol && std::fabs(det - 1.0) <= tol;
}

// parse_trajectory_row (frame_io.cpp:96-115)
void parse_row(const std::string& row, int32_t* frame_index, double* pose12) {
    std::vector<double> fields;
    std::stringstream ss(row);
    std::string token;
    while (std::getline(ss, token, ',')) {
        if (token.empty()) continue;
        try {
            fields.push_back(std::stod(token));
        } catch (const std::exception&) {
            throw Error(SF_IO_ERROR, "trajectory: cannot parse '" + token + "'");
        }
    }
    if (fields.size() != 12 && fields.size() != 13)
        throw Error(SF_IO_ERROR, "trajectory: row needs 12 or 13 comma-separated values");
    size_t k = 0;
    *frame_index = fields.size() == 13 ? static_cast<int32_t>(fields[k++]) : 0;
    m33 R;
    for (int i = 0; i < 9; ++i) R.m[i] = fields[k++];
    if (!is_rotation_host(R, 1e-6)) R = nearest_rotation(R);
    for (int i = 0; i < 9; ++i) pose12[i] = R.m[i];
    for (int i = 0; i < 3; ++i) pose12[9 + i] = fields[k++];
}

}  // namespace

extern "C" {

int sf_trajectory_write(const char* path, const int32_t* frame_index, const double* poses12, uint64_t count) {
    return guarded([&]() -> int {
        if (!path || (count && (!frame_index || !poses12)))
            throw Error(SF_INVALID_ARGUMENT, "sf_trajectory_write: null argument");
        std::ofstream out(path);
        if (!out) throw Error(SF_IO_ERROR, std::string("trajectory: cannot open ") + path + " for writing");
        out << std::setprecision(17);  // frame_io.cpp:84
        for (uint64_t i = 0; i < count; ++i) {
            out << frame_index[i];
            for (int j = 0; j < 12; ++j) out << "," << poses12[12 * i + j];
            out << "\n";
        }
        if (!out) throw Error(SF_IO_ERROR, std::string("trajectory: write failed for ") + path);
        return SF_OK;
    });
}

int sf_trajectory_read(const char* path, int32_t* frame_index, double* poses12, uint64_t* count) {
    return guarded([&]() -> int {
        if (!path || !count) throw Error(SF_INVALID_ARGUMENT, "sf_trajectory_read: null argument");
        std::ifstream in(path);
        if (!in) throw Error(SF_IO_ERROR, std::string("trajectory: cannot open ") + path);
        std::string line;
        uint64_t n = 0;
        const bool fill = frame_index && poses12;
        while (std::getline(in, line)) {
            if (line.empty() || line[0] == '#') continue;  // frame_io.cpp:121
            int32_t fi;
            double p[12];
            parse_row(line, &fi, p);
            if (fill) {
                if (n >= *count) throw Error(SF_OUT_OF_RANGE, "sf_trajectory_read: output capacity");
                frame_index[n] = fi;
                std::memcpy(poses12 + 12 * n, p, sizeof(p));
            }
            ++n;
        }
        *count = n;
        return SF_OK;
    });
}

int sf_dfrm_write(const char* path, const sf_frame* frame) {
    return guarded([&]() -> int {
        if (!path || !frame || !frame->depth) throw Error(SF_INVALID_ARGUMENT, "sf_dfrm_write: null argument");
        const sf_intrinsics& in = frame->intrinsics;
        const size_t n = static_cast<size_t>(in.width) * in.height;
        std::vector<float> depth(n), sigma;
        if (frame->on_device) {
            SF_CUDA(cudaMemcpy(depth.data(), frame->depth, n * sizeof(float), cudaMemcpyDeviceToHost));
        } else {
            std::memcpy(depth.data(), frame->depth, n * sizeof(float));
        }
        if (frame->sigma) {
            sigma.resize(n);
            if (frame->on_device) SF_CUDA(cudaMemcpy(sigma.data(), frame->sigma, n * sizeof(float), cudaMemcpyDeviceToHost));
            else std::memcpy(sigma.data(), frame->sigma, n * sizeof(float));
        }
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Error(SF_IO_ERROR, std::string("dfrm: cannot open ") + path + " for writing");
        out.write("DFRM", 4);
        put_raw<uint32_t>(out, 1u);
        put_raw<uint32_t>(out, static_cast<uint32_t>(in.width));
        put_raw<uint32_t>(out, static_cast<uint32_t>(in.height));
        for (double value : {in.fx, in.fy, in.cx, in.cy, in.near_plane, in.far_plane})
            put_raw<float>(out, static_cast<float>(value));
        out.write(reinterpret_cast<const char*>(depth.data()), static_cast<std::streamsize>(n * sizeof(float)));
        put_raw<uint32_t>(out, frame->sigma ? 1u : 0u);
        if (frame->sigma)
            out.write(reinterpret_cast<const char*>(sigma.data()), static_cast<std::streamsize>(n * sizeof(float)));
        if (!out) throw Error(SF_IO_ERROR, std::string("dfrm: write failed for ") + path);
        return SF_OK;
    });
}

int sf_dfrm_read(const char* path, sf_intrinsics* intrinsics, float* depth, float* sigma, int32_t* has_sigma,
                 int32_t out_on_device) {
    return guarded([&]() -> int {
        if (!path || !intrinsics) throw Error(SF_INVALID_ARGUMENT, "sf_dfrm_read: null argument");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Error(SF_IO_ERROR, std::string("dfrm: cannot open ") + path);
        char magic[4];
        in.read(magic, 4);
        if (!in || std::strncmp(magic, "DFRM", 4) != 0)
            throw Error(SF_IO_ERROR, std::string("dfrm: ") + path + " is not a DFRM file");
        if (get_raw<uint32_t>(in) != 1u) throw Error(SF_IO_ERROR, std::string("dfrm: unsupported version in ") + path);
        sf_intrinsics I{};
        I.width = static_cast<int32_t>(get_raw<uint32_t>(in));
        I.height = static_cast<int32_t>(get_raw<uint32_t>(in));
        I.fx = get_raw<float>(in);
        I.fy = get_raw<float>(in);
        I.cx = get_raw<float>(in);
        I.cy = get_raw<float>(in);
        I.near_plane = get_raw<float>(in);
        I.far_plane = get_raw<float>(in);
        // Intrinsics::validate (camera.cpp:9-14)
        if (I.width <= 0 || I.height <= 0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive image size");
        if (I.fx <= 0.0 || I.fy <= 0.0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive focal length");
        if (!(I.near_plane > 0.0) || !(I.near_plane < I.far_plane))
            throw Error(SF_INVALID_ARGUMENT, "intrinsics: need 0 < near < far");
        *intrinsics = I;
        if (!depth) return SF_OK;  // size query
        const size_t n = static_cast<size_t>(I.width) * I.height;
        std::vector<float> d(n), s;
        in.read(reinterpret_cast<char*>(d.data()), static_cast<std::streamsize>(n * sizeof(float)));
        const bool hs = get_raw<uint32_t>(in) == 1u;
        if (hs) {
            s.resize(n);
            in.read(reinterpret_cast<char*>(s.data()), static_cast<std::streamsize>(n * sizeof(float)));
        }
        if (!in) throw Error(SF_IO_ERROR, std::string("dfrm: truncated file ") + path);
        // out-of-range depths are invalid (frame_io.cpp:75-77)
        for (float& x : d)
            if (x != 0.0f && (x < I.near_plane || x > I.far_plane)) x = 0.0f;
        if (out_on_device) SF_CUDA(cudaMemcpy(depth, d.data(), n * sizeof(float), cudaMemcpyHostToDevice));
        else std::memcpy(depth, d.data(), n * sizeof(float));
        if (has_sigma) *has_sigma = hs ? 1 : 0;
        if (hs && sigma) {
            if (out_on_device) SF_CUDA(cudaMemcpy(sigma, s.data(), n * sizeof(float), cudaMemcpyHostToDevice));
            else std::memcpy(sigma, s.data(), n * sizeof(float));
        }
        return SF_OK;
    });
}

}  // extern "C"
