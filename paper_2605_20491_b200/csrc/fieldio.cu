// Field checkpoint I/O in the reference's binary format (proj/include/kronop/fieldio.hpp:10-13,
// proj/src/fieldio.cpp:28-73): little-endian u32 magic 0x4B4F5046, u32 version 1, u32 dimension,
// u32 scalar kind (0 = f64, 1 = complex f64), u64 extents[dimension], then the raw scalars in
// field order (axis 0 fastest, complex interleaved). Files written here load in the reference and
// vice versa.
//
// Device fields stream through two pinned staging chunks: the device->host copy of chunk i+1
// overlaps the file write of chunk i (and the read of chunk i+1 overlaps the upload of chunk i),
// so an 8 GiB checkpoint costs ~one pass over the file, not file + PCIe back to back.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>

#include "context.cuh"

namespace kronop_dev {

void set_error(const std::string& msg);

namespace {

constexpr uint32_t kMagic = 0x4B4F5046u;
constexpr uint32_t kVersion = 1u;
constexpr size_t kChunkDoubles = size_t(4) << 20;  // 32 MiB staging chunks

template <class F>
int guard_io(F&& f) {
  try {
    f();
    return KRONOP_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return KRONOP_ERUNTIME;
  }
}

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode, const char* what) {
    param_check(path != nullptr, std::string(what) + ": null path");
    f = std::fopen(path, mode);
    param_check(f != nullptr, std::string(what) + ": cannot open " + path);
  }
  ~File() {
    if (f) std::fclose(f);
  }
};

struct Header {
  int d = 0;
  int shape[KRONOP_MAX_DIM] = {};
  int cplx = 0;
  size_t doubles = 0;
};

template <class T>
T read_raw(FILE* f) {
  T v{};
  param_check(std::fread(&v, sizeof(T), 1, f) == 1, "load_field: truncated file");
  return v;
}

Header read_header(FILE* f) {  // fieldio.cpp:51-58
  param_check(read_raw<uint32_t>(f) == kMagic, "load_field: bad magic");
  param_check(read_raw<uint32_t>(f) == kVersion, "load_field: bad version");
  Header h;
  const uint32_t dim = read_raw<uint32_t>(f);
  const uint32_t kind = read_raw<uint32_t>(f);
  param_check(dim >= 1 && dim <= 9, "load_field: bad dimension");
  h.d = static_cast<int>(dim);
  h.doubles = kind == 1 ? 2 : 1;
  for (int a = 0; a < h.d; ++a) {
    const uint64_t n = read_raw<uint64_t>(f);
    param_check(n >= 1 && n <= 0x7fffffffu, "load_field: bad extent");
    h.shape[a] = static_cast<int>(n);
    h.doubles *= n;
  }
  param_check(kind <= 1, "load_field: unknown scalar kind");
  h.cplx = static_cast<int>(kind);
  return h;
}

size_t write_header(FILE* f, int d, const int* shape, int cplx) {  // fieldio.cpp:28-41
  param_check(d >= 1 && d <= KRONOP_MAX_DIM && shape != nullptr,
              "dump_field: dimension must be in [1, 9]");
  const uint32_t head[4] = {kMagic, kVersion, static_cast<uint32_t>(d),
                            static_cast<uint32_t>(cplx ? 1 : 0)};
  param_check(std::fwrite(head, sizeof(head), 1, f) == 1, "dump_field: write failed");
  size_t doubles = cplx ? 2 : 1;
  for (int a = 0; a < d; ++a) {
    param_check(shape[a] >= 1, "dump_field: extents must be positive");
    const uint64_t n = static_cast<uint64_t>(shape[a]);
    param_check(std::fwrite(&n, sizeof(n), 1, f) == 1, "dump_field: write failed");
    doubles *= static_cast<size_t>(shape[a]);
  }
  return doubles;
}

struct Staging {
  double* pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  explicit Staging(size_t n) {
    for (int i = 0; i < 2; ++i) {
      KCUDA(cudaMallocHost(&pin[i], n * sizeof(double)));
      KCUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (pin[i]) cudaFreeHost(pin[i]);
    }
  }
};

}  // namespace

}  // namespace kronop_dev

using namespace kronop_dev;

extern "C" {

int kronop_field_dump_host(const char* path, int d, const int* shape, int is_complex,
                           const double* src) {
  return guard_io([&] {
    File f(path, "wb", "dump_field");
    const size_t n = write_header(f.f, d, shape, is_complex);
    param_check(src != nullptr || n == 0, "dump_field: null data");
    param_check(std::fwrite(src, sizeof(double), n, f.f) == n,
                std::string("dump_field: write failed for ") + path);
  });
}

int kronop_field_load_header(const char* path, int* d, int* shape, int* is_complex) {
  return guard_io([&] {
    param_check(d && shape && is_complex, "load_field: null output");
    File f(path, "rb", "load_field");
    const Header h = read_header(f.f);
    *d = h.d;
    for (int a = 0; a < h.d; ++a) shape[a] = h.shape[a];
    *is_complex = h.cplx;
  });
}

int kronop_field_load_host(const char* path, double* dst, size_t capacity_doubles) {
  return guard_io([&] {
    File f(path, "rb", "load_field");
    const Header h = read_header(f.f);
    param_check(h.doubles <= capacity_doubles, "load_field: destination too small");
    param_check(std::fread(dst, sizeof(double), h.doubles, f.f) == h.doubles,
                "load_field: truncated data");
  });
}

int kronop_field_dump(kronop_ctx* ctx, const char* path, int d, const int* shape, int is_complex,
                      const double* src) {
  return guard_io([&] {
    param_check(ctx != nullptr, "dump_field: null context");
    File f(path, "wb", "dump_field");
    const size_t n = write_header(f.f, d, shape, is_complex);
    param_check(src != nullptr, "dump_field: null data");
    const size_t chunk = n < kChunkDoubles ? n : kChunkDoubles;
    Staging st(chunk);
    const size_t nchunks = (n + chunk - 1) / chunk;
    auto copy_out = [&](size_t c) {
      const size_t off = c * chunk, len = n - off < chunk ? n - off : chunk;
      KCUDA(cudaMemcpyAsync(st.pin[c & 1], src + off, len * sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream));
      KCUDA(cudaEventRecord(st.ev[c & 1], ctx->stream));
    };
    copy_out(0);
    for (size_t c = 0; c < nchunks; ++c) {
      if (c + 1 < nchunks) copy_out(c + 1);  // the other buffer: its previous chunk is written
      KCUDA(cudaEventSynchronize(st.ev[c & 1]));
      const size_t off = c * chunk, len = n - off < chunk ? n - off : chunk;
      param_check(std::fwrite(st.pin[c & 1], sizeof(double), len, f.f) == len,
                  std::string("dump_field: write failed for ") + path);
    }
  });
}

int kronop_field_load(kronop_ctx* ctx, const char* path, double* dst, size_t capacity_doubles) {
  return guard_io([&] {
    param_check(ctx != nullptr && dst != nullptr, "load_field: null argument");
    File f(path, "rb", "load_field");
    const Header h = read_header(f.f);
    param_check(h.doubles <= capacity_doubles, "load_field: destination too small");
    const size_t n = h.doubles;
    const size_t chunk = n < kChunkDoubles ? n : kChunkDoubles;
    Staging st(chunk);
    const size_t nchunks = (n + chunk - 1) / chunk;
    for (size_t c = 0; c < nchunks; ++c) {
      const size_t off = c * chunk, len = n - off < chunk ? n - off : chunk;
      if (c >= 2) KCUDA(cudaEventSynchronize(st.ev[c & 1]));  // upload of chunk c-2 done
      param_check(std::fread(st.pin[c & 1], sizeof(double), len, f.f) == len,
                  "load_field: truncated data");
      KCUDA(cudaMemcpyAsync(dst + off, st.pin[c & 1], len * sizeof(double),
                            cudaMemcpyHostToDevice, ctx->stream));
      KCUDA(cudaEventRecord(st.ev[c & 1], ctx->stream));
    }
    KCUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
