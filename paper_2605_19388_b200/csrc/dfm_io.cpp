// FMNM v2 model container (restates src/io.cpp:49-135): the on-disk format
// for dumped initialisations and fitted models.  Little-endian binary:
//
//   "FMNM" u32 version(=2) u32 bins u32 frames u32 channels u32 sources
//   u32 k_bases u32 n_blocks u32 sizes[n_blocks] u8 shared f64 floor
//   u64 seed f64 sample_rate u32 window_len u32 hop_len u32 iterations
//   u32 n_models
//   per model: T_n (bins x K, col-major) for every n, then V_n (K x frames)
//   Lambda per bin (sources x channels, col-major)
//   W per block, per bin (M_b x M_b complex, col-major)
//
// The payload order is exactly the buffer layout dfm_set_model takes (one
// model), so a dumped init loads straight into a context.  Host code only.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dfm_b200.h"

namespace dfm {
void set_error(const std::string& msg);
}

namespace {

const char kMagic[4] = {'F', 'M', 'N', 'M'};

struct File {
  std::FILE* f = nullptr;
  explicit File(std::FILE* p) : f(p) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

bool layout_ok(const dfm_fmnm_header* h) {
  if (h->n_blocks < 1 || h->n_blocks > DFM_MAX_BLOCKS) return false;
  uint32_t tot = 0;
  for (uint32_t b = 0; b < h->n_blocks; ++b) {
    if (h->sizes[b] < 1 || h->sizes[b] > DFM_MAX_MB) return false;
    tot += h->sizes[b];
  }
  return tot == h->channels;
}

size_t w_count(const dfm_fmnm_header* h) {  // complex values
  size_t n = 0;
  for (uint32_t b = 0; b < h->n_blocks; ++b) n += (size_t)h->num_bins * h->sizes[b] * h->sizes[b];
  return n;
}

}  // namespace

extern "C" {

size_t dfm_fmnm_sizes(const dfm_fmnm_header* h, size_t* n_t, size_t* n_v, size_t* n_lam, size_t* n_w) {
  if (!h) return 0;
  const size_t t = (size_t)h->n_models * h->n_sources * h->num_bins * h->k_bases;
  const size_t v = (size_t)h->n_models * h->n_sources * h->k_bases * h->num_frames;
  const size_t l = (size_t)h->num_bins * h->n_sources * h->channels;
  const size_t w = 2 * w_count(h);
  if (n_t) *n_t = t;
  if (n_v) *n_v = v;
  if (n_lam) *n_lam = l;
  if (n_w) *n_w = w;
  return t + v + l + w;
}

int dfm_fmnm_write(const char* path, const dfm_fmnm_header* h, const double* T, const double* V,
                   const double* lam, const double* w) {
  if (!path || !h || !T || !V || !lam || !w) return DFM_ERR_ARG;
  if (!layout_ok(h)) {
    dfm::set_error("save_model: invalid block layout");
    return DFM_ERR_SHAPE;
  }
  File f(std::fopen(path, "wb"));
  if (!f.f) {
    dfm::set_error(std::string("save_model: cannot open ") + path);
    return DFM_ERR_IO;
  }
  bool ok = std::fwrite(kMagic, 1, 4, f.f) == 4;
  auto put = [&](const void* p, size_t n) { ok = ok && std::fwrite(p, 1, n, f.f) == n; };
  const uint32_t version = DFM_FMNM_VERSION;
  put(&version, 4);
  const uint32_t dims[6] = {h->num_bins, h->num_frames, h->channels, h->n_sources, h->k_bases, h->n_blocks};
  put(dims, sizeof(dims));
  put(h->sizes, 4 * (size_t)h->n_blocks);
  const uint8_t shared = h->shared ? 1 : 0;
  put(&shared, 1);
  put(&h->floor, 8);
  put(&h->seed, 8);
  put(&h->sample_rate, 8);
  const uint32_t tail[4] = {h->window_len, h->hop_len, h->iterations, h->n_models};
  put(tail, sizeof(tail));
  size_t nt, nv, nl, nw;
  dfm_fmnm_sizes(h, &nt, &nv, &nl, &nw);
  // per model: every T_n, then every V_n (io.cpp:76-79)
  const size_t tper = (size_t)h->n_sources * h->num_bins * h->k_bases;
  const size_t vper = (size_t)h->n_sources * h->k_bases * h->num_frames;
  for (uint32_t m = 0; m < h->n_models; ++m) {
    put(T + m * tper, 8 * tper);
    put(V + m * vper, 8 * vper);
  }
  put(lam, 8 * nl);
  put(w, 8 * nw);
  if (!ok) {
    dfm::set_error(std::string("save_model: write failed for ") + path);
    return DFM_ERR_IO;
  }
  return DFM_OK;
}

static int read_impl(const char* path, dfm_fmnm_header* h, double* T, double* V, double* lam, double* w,
                     bool payload) {
  if (!path || !h) return DFM_ERR_ARG;
  File f(std::fopen(path, "rb"));
  if (!f.f) {
    dfm::set_error(std::string("load_model: cannot open ") + path);
    return DFM_ERR_IO;
  }
  bool ok = true;
  auto get = [&](void* p, size_t n) { ok = ok && std::fread(p, 1, n, f.f) == n; };
  char magic[4] = {0, 0, 0, 0};
  get(magic, 4);
  if (!ok || std::memcmp(magic, kMagic, 4) != 0) {
    dfm::set_error(std::string("load_model: bad magic in ") + path);
    return DFM_ERR_IO;
  }
  uint32_t version = 0;
  get(&version, 4);
  if (!ok || version != DFM_FMNM_VERSION) {
    dfm::set_error("load_model: unsupported container version");
    return DFM_ERR_IO;
  }
  std::memset(h, 0, sizeof(*h));
  h->version = version;
  uint32_t dims[6] = {0, 0, 0, 0, 0, 0};
  get(dims, sizeof(dims));
  h->num_bins = dims[0];
  h->num_frames = dims[1];
  h->channels = dims[2];
  h->n_sources = dims[3];
  h->k_bases = dims[4];
  h->n_blocks = dims[5];
  if (!ok || h->n_blocks < 1 || h->n_blocks > DFM_MAX_BLOCKS) {
    dfm::set_error(std::string("load_model: truncated file ") + path);
    return DFM_ERR_IO;
  }
  get(h->sizes, 4 * (size_t)h->n_blocks);
  if (!ok || !layout_ok(h)) {
    dfm::set_error("load_model: layout mismatch");
    return DFM_ERR_IO;
  }
  uint8_t shared = 0;
  get(&shared, 1);
  h->shared = shared != 0;
  get(&h->floor, 8);
  get(&h->seed, 8);
  get(&h->sample_rate, 8);
  uint32_t tail[4] = {0, 0, 0, 0};
  get(tail, sizeof(tail));
  h->window_len = tail[0];
  h->hop_len = tail[1];
  h->iterations = tail[2];
  h->n_models = tail[3];
  if (!ok) {
    dfm::set_error(std::string("load_model: truncated file ") + path);
    return DFM_ERR_IO;
  }
  if (!payload) return DFM_OK;
  if (!T || !V || !lam || !w) return DFM_ERR_ARG;
  size_t nt, nv, nl, nw;
  dfm_fmnm_sizes(h, &nt, &nv, &nl, &nw);
  const size_t tper = (size_t)h->n_sources * h->num_bins * h->k_bases;
  const size_t vper = (size_t)h->n_sources * h->k_bases * h->num_frames;
  for (uint32_t m = 0; m < h->n_models; ++m) {
    get(T + m * tper, 8 * tper);
    get(V + m * vper, 8 * vper);
  }
  get(lam, 8 * nl);
  get(w, 8 * nw);
  if (!ok) {
    dfm::set_error(std::string("load_model: truncated file ") + path);
    return DFM_ERR_IO;
  }
  return DFM_OK;
}

int dfm_fmnm_read_header(const char* path, dfm_fmnm_header* h) {
  return read_impl(path, h, nullptr, nullptr, nullptr, nullptr, false);
}

int dfm_fmnm_read(const char* path, dfm_fmnm_header* h, double* T, double* V, double* lam, double* w) {
  return read_impl(path, h, T, V, lam, w, true);
}

}  // extern "C"
