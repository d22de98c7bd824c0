// Dataset harness and dataset comparison (row f4) over
// the B200 path: dataset::run_press_dataset / compare_datasets and the
// manifest CSV (/root/reference/proj/src/dataset/harness.cpp:55-245,
// include/tacchi/dataset/harness.hpp:14-66).
//
// B200 shape of the reference's thread pool (harness.cpp:206-237): the
// (object, position) jobs run as a batch of independent device simulations
// stepped together (tg_step_many submits every handle's substep graph before
// waiting), captured on device at the schedule's substeps, and the PNG /
// .depth encoding runs on a host writer pool while the GPU keeps stepping.
// Every output file, the manifest and config.json have the reference's names
// and formats; the manifest is rewritten sorted, so runs are reproducible.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <deque>
#include <exception>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <numeric>
#include <cstring>
#include <cstdlib>
#include <iterator>
#include <stdexcept>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "host_config.hpp"
#include "tacchi_cuda.h"

namespace tacchi_b200 {
int fail(int code, const std::string& msg);
}

namespace tacchi_b200::dataset {

namespace fs = std::filesystem;
using host::Config;
using host::HostError;
using host::V3;

namespace {

void check(int rc) {
  if (rc != TG_OK) throw HostError{rc, tg_last_error()};
}

}  // namespace

// harness.hpp:14-25
struct ManifestRow {
  std::string object;
  int position_index = 0;
  double pos_x_mm = 0.0, pos_y_mm = 0.0;
  int depth_index = 0;
  double depth_mm = 0.0;
  bool contact = false;
  uint64_t particle_count = 0;
  std::string image, depth_map;
};

namespace {

// (object, position, depth level): the identity of a manifest row.
using RowKey = std::tuple<std::string, int, int>;
RowKey key_of(const ManifestRow& r) { return {r.object, r.position_index, r.depth_index}; }

// Output file stem of a row: <object>_pNN_dNN (harness.cpp:75-94 names).
std::string file_stem(const std::string& object, int position, int depth) {
  std::string out = object;
  char tail[24];
  std::snprintf(tail, sizeof(tail), "_p%02d_d%02d", position, depth);
  return out.append(tail);
}

// Strict field conversions of a manifest cell (the whole cell must parse).
long long cell_int(const std::string& c) {
  char* end = nullptr;
  const long long v = std::strtoll(c.c_str(), &end, 10);
  if (c.empty() || *end != '\0') throw std::invalid_argument(c);
  return v;
}
double cell_real(const std::string& c) {
  char* end = nullptr;
  const double v = std::strtod(c.c_str(), &end);
  if (c.empty() || *end != '\0') throw std::invalid_argument(c);
  return v;
}

// Mean and sample standard deviation (n - 1), two passes left to right.
struct Moments {
  double mean = 0.0, stdev = 0.0;
};
Moments moments(const std::vector<double>& xs) {
  Moments m;
  if (xs.empty()) return m;
  m.mean = std::accumulate(xs.begin(), xs.end(), 0.0) / static_cast<double>(xs.size());
  if (xs.size() > 1) {
    double ss = 0.0;
    for (double x : xs) ss += (x - m.mean) * (x - m.mean);
    m.stdev = std::sqrt(ss / static_cast<double>(xs.size() - 1));
  }
  return m;
}

// A small FIFO pool for host file encoding (PNG deflate dominates).
class WriterPool {
 public:
  explicit WriterPool(int n) {
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~WriterPool() { finish(); }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(m_);
      q_.push_back(std::move(f));
    }
    cv_.notify_one();
  }
  // Drains the queue, joins the threads and rethrows the first failure.
  void finish() {
    {
      std::lock_guard<std::mutex> lk(m_);
      done_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_)
      if (t.joinable()) t.join();
    threads_.clear();
    if (error_) {
      auto e = error_;
      error_ = nullptr;
      std::rethrow_exception(e);
    }
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [this] { return done_ || !q_.empty(); });
        if (q_.empty()) return;
        f = std::move(q_.front());
        q_.pop_front();
      }
      try {
        f();
      } catch (...) {
        std::lock_guard<std::mutex> lk(m_);
        if (!error_) error_ = std::current_exception();
      }
    }
  }
  std::vector<std::thread> threads_;
  std::deque<std::function<void()>> q_;
  std::mutex m_;
  std::condition_variable cv_;
  bool done_ = false;
  std::exception_ptr error_;
};

// One object's indenter cloud, shared by its positions: sampled on the
// device for a generated shape (f3), else generated / loaded on the host.
struct ObjectCloud {
  std::shared_ptr<host::DeviceCloud> dev;
  std::vector<V3> host;
  size_t size() const { return dev ? host::device_cloud_size(*dev) : host.size(); }
};

struct PositionJob {
  std::string object;
  std::shared_ptr<ObjectCloud> cloud;
  int position_index;
  double offset_x_m, offset_y_m;
};

struct Handle {
  tg_handle h = nullptr;
  ~Handle() {
    if (h) tg_destroy(h);
  }
};

int writer_threads() {
  const unsigned hc = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(2u, std::min(16u, hc ? hc : 4u)));
}

}  // namespace

// The manifest CSV (harness.cpp:114-157): a header line, then one row per
// capture, ten comma-separated cells (no quoting: names never hold commas).
std::vector<ManifestRow> read_manifest(const fs::path& csv_path) {
  std::ifstream in(csv_path);
  if (!in) throw HostError{TG_ERR_IO, "cannot open manifest " + csv_path.string()};
  const auto malformed = [&] {
    return HostError{TG_ERR_PARSE, csv_path.string() + ": malformed manifest row"};
  };
  std::vector<ManifestRow> rows;
  std::string text;
  bool seen_header = false;
  while (std::getline(in, text)) {
    if (text.empty()) continue;
    if (!seen_header) {  // the first non-empty line is the header
      seen_header = true;
      continue;
    }
    std::vector<std::string> cell(1);
    for (char ch : text) {
      if (ch == ',') cell.emplace_back();
      else cell.back().push_back(ch);
    }
    if (!cell.empty() && cell.back().empty() && text.back() == ',') cell.pop_back();
    if (cell.size() != 10) throw malformed();
    ManifestRow r;
    try {
      r.position_index = static_cast<int>(cell_int(cell[1]));
      r.pos_x_mm = cell_real(cell[2]);
      r.pos_y_mm = cell_real(cell[3]);
      r.depth_index = static_cast<int>(cell_int(cell[4]));
      r.depth_mm = cell_real(cell[5]);
      r.particle_count = static_cast<uint64_t>(cell_int(cell[7]));
    } catch (const std::exception&) {
      throw malformed();
    }
    r.object = std::move(cell[0]);
    r.contact = cell[6] == "1" || cell[6] == "true";
    r.image = std::move(cell[8]);
    r.depth_map = std::move(cell[9]);
    rows.push_back(std::move(r));
  }
  return rows;
}

void write_manifest(const std::vector<ManifestRow>& rows, const fs::path& csv_path) {
  std::string body =
      "object,position_index,pos_x_mm,pos_y_mm,depth_index,depth_mm,contact,"
      "particle_count,image,depth_map\n";
  for (const ManifestRow& r : rows) {
    char nums[160];
    std::snprintf(nums, sizeof(nums), ",%d,%.6g,%.6g,%d,%.6g,%d,%llu,", r.position_index,
                  r.pos_x_mm, r.pos_y_mm, r.depth_index, r.depth_mm, r.contact ? 1 : 0,
                  static_cast<unsigned long long>(r.particle_count));
    body += r.object;
    body += nums;
    body += r.image;
    body += ',';
    body += r.depth_map;
    body += '\n';
  }
  std::ofstream out(csv_path, std::ios::binary | std::ios::trunc);
  if (!out) throw HostError{TG_ERR_IO, "cannot write manifest " + csv_path.string()};
  out << body;
}

// Resume (harness.cpp:166-179): the rows of (object, position) groups whose
// every depth level is present are kept, and those groups are not re-run.
struct ResumeState {
  std::vector<ManifestRow> kept;
  std::set<std::pair<std::string, int>> complete;
};
ResumeState resume_from(const fs::path& manifest_path, size_t levels) {
  ResumeState st;
  if (!fs::exists(manifest_path)) return st;
  std::vector<ManifestRow> prior = read_manifest(manifest_path);
  std::map<std::pair<std::string, int>, std::set<int>> levels_of;
  for (const ManifestRow& r : prior) levels_of[{r.object, r.position_index}].insert(r.depth_index);
  for (const auto& entry : levels_of)
    if (entry.second.size() == levels) st.complete.insert(entry.first);
  std::copy_if(prior.begin(), prior.end(), std::back_inserter(st.kept), [&](const ManifestRow& r) {
    return st.complete.count({r.object, r.position_index}) > 0;
  });
  return st;
}

struct DatasetResult {
  size_t rows = 0, skipped_positions = 0;
};

// run_press_dataset (harness.cpp:159-245) with run_position (:55-103) batched
// on the device. `batch` = simulations stepped together (0: config workers,
// else 16).
DatasetResult run_press_dataset(const std::string& cfg_json, const fs::path& out_dir, int device,
                                int batch) {
  const Config cfg = host::parse_config(cfg_json.c_str());
  host::validate(cfg);
  fs::create_directories(out_dir / "images");
  fs::create_directories(out_dir / "depth");
  {
    std::ofstream out(out_dir / "config.json");
    if (!out) throw HostError{TG_ERR_IO, "cannot write " + (out_dir / "config.json").string()};
    out << host::to_json_string(cfg);
  }

  const fs::path manifest_path = out_dir / "manifest.csv";
  ResumeState resume = resume_from(manifest_path, cfg.depths_mm.size());
  std::vector<ManifestRow>& kept = resume.kept;
  const auto& done = resume.complete;

  // Jobs: every object at every press-grid position; one cloud per object
  // (harness.cpp:194-195 shares it across positions): generated shapes are
  // sampled on the device, point-cloud files are read on host threads.
  const double step_m = cfg.step_mm * 1e-3;
  std::vector<PositionJob> jobs;
  size_t skipped = 0;
  std::map<std::string, std::shared_ptr<ObjectCloud>> clouds;
  for (const std::string& object : cfg.objects)
    for (int py = 0; py < cfg.positions_y; ++py)
      for (int px = 0; px < cfg.positions_x; ++px) {
        const int index = py * cfg.positions_x + px;
        if (done.count({object, index})) {
          ++skipped;
          continue;
        }
        auto& cloud = clouds[object];
        if (!cloud) cloud = std::make_shared<ObjectCloud>();
        jobs.push_back({object, cloud, index, (px - 0.5 * (cfg.positions_x - 1)) * step_m,
                        (py - 0.5 * (cfg.positions_y - 1)) * step_m});
      }
  {
    std::vector<std::thread> gen;
    std::vector<std::exception_ptr> errs(clouds.size());
    size_t k = 0;
    for (auto& [object, cloud] : clouds) {
      cloud->dev = host::device_cloud_for_object(device, cfg, object);
      if (!cloud->dev)
        gen.emplace_back([&cfg, object = object, cloud = cloud, &errs, k] {
          try {
            cloud->host = host::indenter_cloud_for(cfg, object);
          } catch (...) {
            errs[k] = std::current_exception();
          }
        });
      ++k;
    }
    for (auto& t : gen) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }

  // Substep index at which the commanded depth crosses each level.
  const double v = cfg.press_speed_mm_s * 1e-3;
  const double gap = cfg.gap_mm * 1e-3;
  const double per_step = v * cfg.dt;
  std::map<int64_t, std::vector<int>> schedule;
  for (size_t k = 0; k < cfg.depths_mm.size(); ++k) {
    const double travel = gap + cfg.depths_mm[k] * 1e-3;
    schedule[static_cast<int64_t>(std::llround(travel / per_step))].push_back(static_cast<int>(k));
  }

  if (batch <= 0) batch = cfg.workers > 0 ? cfg.workers : 16;
  batch = std::max(1, std::min<int>(batch, static_cast<int>(jobs.size())));

  std::vector<ManifestRow> fresh;
  std::mutex rows_mutex;
  WriterPool writers(writer_threads());
  std::map<std::string, tg_render> renders;
  for (const auto& [object, cloud] : clouds) {
    tg_render r{};
    check(tg_render_from_config(cfg_json.c_str(), object.c_str(), &r));
    renders[object] = r;
  }

  try {
    for (size_t b0 = 0; b0 < jobs.size(); b0 += batch) {
      const size_t nb = std::min(jobs.size() - b0, static_cast<size_t>(batch));
      std::vector<Handle> sims(nb);
      std::vector<tg_handle> hs(nb);
      for (size_t i = 0; i < nb; ++i) {
        const PositionJob& job = jobs[b0 + i];
        const std::vector<V3> placed =
            job.cloud->dev
                ? host::place_for_press_on(*job.cloud->dev, cfg, job.offset_x_m, job.offset_y_m)
                : host::place_for_press(cfg, job.cloud->host, job.offset_x_m, job.offset_y_m);
        check(host::build_sim_from(device, cfg, placed, &sims[i].h));
        hs[i] = sims[i].h;
      }
      std::vector<double> vel(3 * nb);
      for (size_t i = 0; i < nb; ++i) {
        vel[3 * i] = 0.0;
        vel[3 * i + 1] = 0.0;
        vel[3 * i + 2] = -v;
      }
      // The chunk that reaches a capture level is submitted together with
      // every handle's capture (tg_step_capture_many: one wait per handle).
      std::vector<tg_render> rs(nb);
      for (size_t i = 0; i < nb; ++i) rs[i] = renders.at(jobs[b0 + i].object);
      auto step_and_capture = [&](int n, const std::vector<int>& levels) {
        std::vector<std::shared_ptr<std::vector<double>>> depth(nb);
        std::vector<std::shared_ptr<std::vector<uint8_t>>> rgb(nb);
        std::vector<double*> dp(nb);
        std::vector<uint8_t*> cp(nb);
        for (size_t i = 0; i < nb; ++i) {
          const size_t px = static_cast<size_t>(rs[i].width) * rs[i].height;
          depth[i] = std::make_shared<std::vector<double>>(px);
          rgb[i] = std::make_shared<std::vector<uint8_t>>(px * 3);
          dp[i] = depth[i]->data();
          cp[i] = rgb[i]->data();
        }
        check(tg_step_capture_many(hs.data(), static_cast<int>(nb), vel.data(), n, rs.data(),
                                   static_cast<int>(nb), dp.data(), cp.data(), nullptr));
        for (size_t i = 0; i < nb; ++i) {
          const PositionJob& job = jobs[b0 + i];
          const tg_render& r = rs[i];
          for (int k : levels) {
            ManifestRow row;
            row.object = job.object;
            row.position_index = job.position_index;
            row.pos_x_mm = job.offset_x_m * 1e3;
            row.pos_y_mm = job.offset_y_m * 1e3;
            row.depth_index = k;
            row.depth_mm = cfg.depths_mm[k];
            row.contact = cfg.depths_mm[k] > 0.0;
            row.particle_count = job.cloud->size();
            const std::string stem = file_stem(job.object, job.position_index, k);
            row.image = "images/" + stem + ".png";
            row.depth_map = "depth/" + stem + ".depth";
            const std::string png = (out_dir / row.image).string();
            const std::string dep = (out_dir / row.depth_map).string();
            const int w = r.width, h = r.height;
            const double ptm = r.pixel_to_meter * r.crop_scale;
            writers.submit([png, dep, w, h, ptm, d = depth[i], c = rgb[i]] {
              host::save_png(png, w, h, c->data());
              host::save_depth_map(dep, w, h, ptm, d->data());
            });
            std::lock_guard<std::mutex> lk(rows_mutex);
            fresh.push_back(std::move(row));
          }
        }
      };
      int64_t cur = 0;
      for (const auto& [s, levels] : schedule) {
        while (s - cur > 200) {
          check(tg_step_many(hs.data(), static_cast<int>(nb), vel.data(), 200));
          cur += 200;
        }
        step_and_capture(static_cast<int>(s - cur), levels);
        cur = s;
      }
    }
  } catch (...) {
    try {
      writers.finish();
    } catch (...) {
    }
    throw;
  }
  writers.finish();

  std::vector<ManifestRow> all = std::move(kept);
  for (auto& r : fresh) all.push_back(std::move(r));
  std::sort(all.begin(), all.end(),
            [](const ManifestRow& a, const ManifestRow& b) { return key_of(a) < key_of(b); });
  write_manifest(all, manifest_path);
  return {all.size(), skipped};
}

struct CompareAggregate {
  size_t pairs = 0;
  double ssim_mean = 0, ssim_std = 0, psnr_mean = 0, psnr_std = 0, mae_mean = 0, mae_std = 0;
};

// compare_datasets (harness.cpp:247-321). The keys of both manifests must
// match; the image pairs are then evaluated in chunks of kChunk: the chunk's
// PNGs are decoded on host threads into one pair-major staging buffer per
// side, scored with one batched device launch (tg_image_metrics), and
// released before the next chunk, so host memory stays bounded for any
// dataset size.
CompareAggregate compare_datasets(const fs::path& dir_a, const fs::path& dir_b,
                                  const fs::path& csv_out, int device) {
  std::map<RowKey, ManifestRow> side_a, side_b;
  for (auto& r : read_manifest(dir_a / "manifest.csv")) side_a.emplace(key_of(r), std::move(r));
  for (auto& r : read_manifest(dir_b / "manifest.csv")) side_b.emplace(key_of(r), std::move(r));

  // Keys present on one side only (first eight named in the message).
  std::vector<std::pair<RowKey, const char*>> absent;
  for (const auto& [k, r] : side_a)
    if (!side_b.count(k)) absent.emplace_back(k, "B");
  for (const auto& [k, r] : side_b)
    if (!side_a.count(k)) absent.emplace_back(k, "A");
  if (!absent.empty()) {
    std::string detail;
    for (size_t i = 0; i < absent.size() && i < 8; ++i) {
      const RowKey& k = absent[i].first;
      if (i) detail += "; ";
      detail += std::get<0>(k) + "/p" + std::to_string(std::get<1>(k)) + "/d" +
                std::to_string(std::get<2>(k)) + " missing in " + absent[i].second;
    }
    throw HostError{TG_ERR_MANIFEST_MISMATCH,
                    "manifests differ (" + std::to_string(absent.size()) + " keys): " + detail};
  }

  std::vector<RowKey> keys;
  keys.reserve(side_a.size());
  for (const auto& entry : side_a) keys.push_back(entry.first);
  const size_t n = keys.size();
  std::vector<double> ssim(n), psnr(n), mae(n);
  constexpr size_t kChunk = 256;
  const int threads = writer_threads();
  for (size_t c0 = 0; c0 < n; c0 += kChunk) {
    const size_t cn = std::min(kChunk, n - c0);
    std::vector<std::vector<uint8_t>> img(2 * cn);
    std::vector<int> w(2 * cn), h(2 * cn);
    std::vector<std::exception_ptr> err(2 * cn);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        for (size_t j = t; j < 2 * cn; j += threads) {
          const RowKey& k = keys[c0 + j / 2];
          const fs::path path = (j & 1) ? dir_b / side_b.at(k).image : dir_a / side_a.at(k).image;
          try {
            img[j] = host::load_png(path.string(), w[j], h[j]);
          } catch (...) {
            err[j] = std::current_exception();
          }
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
    // runs of pairs that share one image size go to the device together
    for (size_t j0 = 0; j0 < cn;) {
      const int W = w[2 * j0], H = h[2 * j0];
      if (w[2 * j0 + 1] != W || h[2 * j0 + 1] != H)
        throw HostError{TG_ERR_SHAPE_MISMATCH, "image shapes differ: " + std::to_string(W) + "x" +
                                                   std::to_string(H) + " vs " +
                                                   std::to_string(w[2 * j0 + 1]) + "x" +
                                                   std::to_string(h[2 * j0 + 1])};
      size_t j1 = j0 + 1;
      while (j1 < cn && w[2 * j1] == W && h[2 * j1] == H && w[2 * j1 + 1] == W && h[2 * j1 + 1] == H)
        ++j1;
      const size_t bytes = static_cast<size_t>(W) * H * 3;
      std::vector<uint8_t> A(bytes * (j1 - j0)), B(bytes * (j1 - j0));
      for (size_t j = j0; j < j1; ++j) {
        std::memcpy(A.data() + (j - j0) * bytes, img[2 * j].data(), bytes);
        std::memcpy(B.data() + (j - j0) * bytes, img[2 * j + 1].data(), bytes);
        img[2 * j].clear();
        img[2 * j].shrink_to_fit();
        img[2 * j + 1].clear();
        img[2 * j + 1].shrink_to_fit();
      }
      std::vector<double> m(3 * (j1 - j0));
      check(tg_image_metrics(device, A.data(), B.data(), W, H, static_cast<int>(j1 - j0), m.data()));
      for (size_t j = j0; j < j1; ++j) {
        ssim[c0 + j] = m[3 * (j - j0)];
        psnr[c0 + j] = m[3 * (j - j0) + 1];
        mae[c0 + j] = m[3 * (j - j0) + 2];
      }
      j0 = j1;
    }
  }

  CompareAggregate agg;
  agg.pairs = n;
  const Moments ms = moments(ssim), mp = moments(psnr), mm = moments(mae);
  agg.ssim_mean = ms.mean;
  agg.ssim_std = ms.stdev;
  agg.psnr_mean = mp.mean;
  agg.psnr_std = mp.stdev;
  agg.mae_mean = mm.mean;
  agg.mae_std = mm.stdev;
  if (!csv_out.empty()) {
    std::ofstream csv(csv_out, std::ios::binary | std::ios::trunc);
    if (!csv) throw HostError{TG_ERR_IO, "cannot write " + csv_out.string()};
    char line[512];
    csv << "object,position_index,depth_index,ssim,psnr_db,mae_pct\n";
    for (size_t i = 0; i < n; ++i) {
      std::snprintf(line, sizeof(line), ",%d,%d,%.6f,%.4f,%.4f\n", std::get<1>(keys[i]),
                    std::get<2>(keys[i]), ssim[i], psnr[i], mae[i]);
      csv << std::get<0>(keys[i]) << line;
    }
    std::snprintf(line, sizeof(line), "mean,,,%.6f,%.4f,%.4f\nstd,,,%.6f,%.4f,%.4f\n",
                  agg.ssim_mean, agg.psnr_mean, agg.mae_mean, agg.ssim_std, agg.psnr_std,
                  agg.mae_std);
    csv << line;
  }
  return agg;
}

}  // namespace tacchi_b200::dataset

extern "C" {

int tg_run_press_dataset(int device, const char* config_json, const char* out_dir, int batch,
                         int64_t* rows, int64_t* skipped_positions) {
  try {
    const auto r = tacchi_b200::dataset::run_press_dataset(config_json ? config_json : "",
                                                           out_dir ? out_dir : ".", device, batch);
    if (rows) *rows = static_cast<int64_t>(r.rows);
    if (skipped_positions) *skipped_positions = static_cast<int64_t>(r.skipped_positions);
    return TG_OK;
  } catch (const tacchi_b200::host::HostError& e) {
    return tacchi_b200::fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return tacchi_b200::fail(TG_ERR_IO, e.what());
  }
}

int tg_compare_datasets(int device, const char* dir_a, const char* dir_b, const char* csv_out,
                        double* out) {
  try {
    const auto a = tacchi_b200::dataset::compare_datasets(dir_a ? dir_a : "", dir_b ? dir_b : "",
                                                          csv_out ? csv_out : "", device);
    if (out) {
      out[0] = static_cast<double>(a.pairs);
      out[1] = a.ssim_mean;
      out[2] = a.ssim_std;
      out[3] = a.psnr_mean;
      out[4] = a.psnr_std;
      out[5] = a.mae_mean;
      out[6] = a.mae_std;
    }
    return TG_OK;
  } catch (const tacchi_b200::host::HostError& e) {
    return tacchi_b200::fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return tacchi_b200::fail(TG_ERR_IO, e.what());
  }
}

int tg_load_png(const char* path, uint8_t* rgb, int* w, int* h) {
  try {
    int ww = 0, hh = 0;
    const auto img = tacchi_b200::host::load_png(path ? path : "", ww, hh);
    if (w) *w = ww;
    if (h) *h = hh;
    if (rgb) std::copy(img.begin(), img.end(), rgb);
    return TG_OK;
  } catch (const tacchi_b200::host::HostError& e) {
    return tacchi_b200::fail(e.code, e.msg);
  }
}

int tg_save_png(const char* path, const uint8_t* rgb, int w, int h) {
  try {
    if (w <= 0 || h <= 0) throw tacchi_b200::host::HostError{TG_ERR_IO, "save_png: empty image"};
    tacchi_b200::host::save_png(path ? path : "", w, h, rgb);
    return TG_OK;
  } catch (const tacchi_b200::host::HostError& e) {
    return tacchi_b200::fail(e.code, e.msg);
  }
}

}  // extern "C"
