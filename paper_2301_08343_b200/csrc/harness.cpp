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

std::string row_file_stem(const std::string& object, int position, int depth) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "_p%02d_d%02d", position, depth);
  return object + buf;
}

std::vector<std::string> split_csv_line(const std::string& line) {
  std::vector<std::string> out;
  std::stringstream ss(line);
  std::string field;
  while (std::getline(ss, field, ',')) out.push_back(field);
  return out;
}

bool row_key_less(const ManifestRow& a, const ManifestRow& b) {
  return std::tie(a.object, a.position_index, a.depth_index) <
         std::tie(b.object, b.position_index, b.depth_index);
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

struct PositionJob {
  std::string object;
  std::shared_ptr<const std::vector<V3>> cloud;
  int position_index;
  double offset_x_m, offset_y_m;
};

struct Handle {
  tg_handle h = nullptr;
  ~Handle() {
    if (h) tg_destroy(h);
  }
};

double aggregate_std(const std::vector<double>& xs, double mean) {
  if (xs.size() < 2) return 0.0;
  double acc = 0.0;
  for (double x : xs) acc += (x - mean) * (x - mean);
  return std::sqrt(acc / static_cast<double>(xs.size() - 1));
}

int writer_threads() {
  const unsigned hc = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(2u, std::min(16u, hc ? hc : 4u)));
}

}  // namespace

// harness.cpp:114-142
std::vector<ManifestRow> read_manifest(const fs::path& csv_path) {
  std::ifstream in(csv_path);
  if (!in) throw HostError{TG_ERR_IO, "cannot open manifest " + csv_path.string()};
  std::vector<ManifestRow> rows;
  std::string line;
  bool header = true;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    if (header) {
      header = false;
      continue;
    }
    const auto f = split_csv_line(line);
    if (f.size() != 10) throw HostError{TG_ERR_PARSE, csv_path.string() + ": malformed manifest row"};
    ManifestRow r;
    try {
      r.object = f[0];
      r.position_index = std::stoi(f[1]);
      r.pos_x_mm = std::stod(f[2]);
      r.pos_y_mm = std::stod(f[3]);
      r.depth_index = std::stoi(f[4]);
      r.depth_mm = std::stod(f[5]);
      r.contact = f[6] == "1" || f[6] == "true";
      r.particle_count = std::stoull(f[7]);
    } catch (const std::exception&) {
      throw HostError{TG_ERR_PARSE, csv_path.string() + ": malformed manifest row"};
    }
    r.image = f[8];
    r.depth_map = f[9];
    rows.push_back(std::move(r));
  }
  return rows;
}

// harness.cpp:144-157
void write_manifest(const std::vector<ManifestRow>& rows, const fs::path& csv_path) {
  std::FILE* f = std::fopen(csv_path.string().c_str(), "w");
  if (!f) throw HostError{TG_ERR_IO, "cannot write manifest " + csv_path.string()};
  std::fprintf(f,
               "object,position_index,pos_x_mm,pos_y_mm,depth_index,depth_mm,contact,"
               "particle_count,image,depth_map\n");
  for (const ManifestRow& r : rows)
    std::fprintf(f, "%s,%d,%.6g,%.6g,%d,%.6g,%d,%llu,%s,%s\n", r.object.c_str(), r.position_index,
                 r.pos_x_mm, r.pos_y_mm, r.depth_index, r.depth_mm, r.contact ? 1 : 0,
                 static_cast<unsigned long long>(r.particle_count), r.image.c_str(),
                 r.depth_map.c_str());
  std::fclose(f);
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

  // Resume: keep rows of (object, position) groups that are already complete.
  std::vector<ManifestRow> kept;
  std::set<std::pair<std::string, int>> done;
  const fs::path manifest_path = out_dir / "manifest.csv";
  if (fs::exists(manifest_path)) {
    std::map<std::pair<std::string, int>, std::set<int>> seen;
    const auto existing = read_manifest(manifest_path);
    for (const ManifestRow& r : existing) seen[{r.object, r.position_index}].insert(r.depth_index);
    for (const auto& [key, depths] : seen)
      if (depths.size() == cfg.depths_mm.size()) done.insert(key);
    for (const ManifestRow& r : existing)
      if (done.count({r.object, r.position_index})) kept.push_back(r);
  }

  // Jobs: every object at every press-grid position; one cloud per object,
  // generated on host threads in parallel (rejection sampling of 1e6 points
  // per object, harness.cpp:194-195 shares it across positions).
  const double step_m = cfg.step_mm * 1e-3;
  std::vector<PositionJob> jobs;
  size_t skipped = 0;
  std::map<std::string, std::shared_ptr<std::vector<V3>>> clouds;
  for (const std::string& object : cfg.objects)
    for (int py = 0; py < cfg.positions_y; ++py)
      for (int px = 0; px < cfg.positions_x; ++px) {
        const int index = py * cfg.positions_x + px;
        if (done.count({object, index})) {
          ++skipped;
          continue;
        }
        auto& cloud = clouds[object];
        if (!cloud) cloud = std::make_shared<std::vector<V3>>();
        jobs.push_back({object, cloud, index, (px - 0.5 * (cfg.positions_x - 1)) * step_m,
                        (py - 0.5 * (cfg.positions_y - 1)) * step_m});
      }
  {
    std::vector<std::thread> gen;
    std::vector<std::exception_ptr> errs(clouds.size());
    size_t k = 0;
    for (auto& [object, cloud] : clouds) {
      gen.emplace_back([&cfg, object = object, cloud = cloud, &errs, k] {
        try {
          *cloud = host::indenter_cloud_for(cfg, object);
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
            host::place_for_press(cfg, *job.cloud, job.offset_x_m, job.offset_y_m);
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
            const std::string stem = row_file_stem(job.object, job.position_index, k);
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
  std::sort(all.begin(), all.end(), row_key_less);
  write_manifest(all, manifest_path);
  return {all.size(), skipped};
}

int image_metrics_batch(int device, const std::vector<std::vector<uint8_t>>& a,
                        const std::vector<std::vector<uint8_t>>& b, int w, int h,
                        std::vector<double>& out) {
  const size_t n = a.size(), px = static_cast<size_t>(w) * h * 3;
  std::vector<uint8_t> ha(n * px), hb(n * px);
  for (size_t i = 0; i < n; ++i) {
    std::copy(a[i].begin(), a[i].end(), ha.begin() + i * px);
    std::copy(b[i].begin(), b[i].end(), hb.begin() + i * px);
  }
  out.assign(3 * n, 0.0);
  return tg_image_metrics(device, ha.data(), hb.data(), w, h, static_cast<int>(n), out.data());
}

struct CompareAggregate {
  size_t pairs = 0;
  double ssim_mean = 0, ssim_std = 0, psnr_mean = 0, psnr_std = 0, mae_mean = 0, mae_std = 0;
};

// compare_datasets (harness.cpp:247-321): PNG decode on host threads, the
// metrics for every pair of one image size in batched device launches.
CompareAggregate compare_datasets(const fs::path& dir_a, const fs::path& dir_b,
                                  const fs::path& csv_out, int device) {
  const auto rows_a = read_manifest(dir_a / "manifest.csv");
  const auto rows_b = read_manifest(dir_b / "manifest.csv");
  using Key = std::tuple<std::string, int, int>;
  std::map<Key, const ManifestRow*> map_a, map_b;
  for (const auto& r : rows_b) map_b[{r.object, r.position_index, r.depth_index}] = &r;
  for (const auto& r : rows_a) map_a[{r.object, r.position_index, r.depth_index}] = &r;

  std::string missing;
  int missing_count = 0;
  auto note_missing = [&](const Key& k, const char* side) {
    if (missing_count++ < 8)
      missing += std::string(missing.empty() ? "" : "; ") + std::get<0>(k) + "/p" +
                 std::to_string(std::get<1>(k)) + "/d" + std::to_string(std::get<2>(k)) +
                 " missing in " + side;
  };
  for (const auto& [k, r] : map_a)
    if (!map_b.count(k)) note_missing(k, "B");
  for (const auto& [k, r] : map_b)
    if (!map_a.count(k)) note_missing(k, "A");
  if (missing_count > 0)
    throw HostError{TG_ERR_MANIFEST_MISMATCH, "manifests differ (" + std::to_string(missing_count) +
                                                  " keys): " + missing};

  std::vector<Key> keys;
  for (const auto& [k, r] : map_a) keys.push_back(k);
  const size_t n = keys.size();
  std::vector<std::vector<uint8_t>> ia(n), ib(n);
  std::vector<int> wa(n), ha(n), wb(n), hb(n);
  {
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(n);
    const int nt = writer_threads();
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (size_t i = t; i < n; i += nt) {
          try {
            ia[i] = host::load_png((dir_a / map_a.at(keys[i])->image).string(), wa[i], ha[i]);
            ib[i] = host::load_png((dir_b / map_b.at(keys[i])->image).string(), wb[i], hb[i]);
          } catch (...) {
            errs[i] = std::current_exception();
          }
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  std::vector<double> ssims(n), psnrs(n), maes(n);
  // Batch consecutive pairs of one shape (all of them for a real dataset).
  for (size_t i0 = 0; i0 < n;) {
    if (wa[i0] != wb[i0] || ha[i0] != hb[i0])
      throw HostError{TG_ERR_SHAPE_MISMATCH,
                      "image shapes differ: " + std::to_string(wa[i0]) + "x" + std::to_string(ha[i0]) +
                          " vs " + std::to_string(wb[i0]) + "x" + std::to_string(hb[i0])};
    size_t i1 = i0 + 1;
    while (i1 < n && i1 - i0 < 256 && wa[i1] == wa[i0] && ha[i1] == ha[i0] && wb[i1] == wa[i0] &&
           hb[i1] == ha[i0])
      ++i1;
    std::vector<std::vector<uint8_t>> A(ia.begin() + i0, ia.begin() + i1),
        B(ib.begin() + i0, ib.begin() + i1);
    std::vector<double> m;
    check(image_metrics_batch(device, A, B, wa[i0], ha[i0], m));
    for (size_t i = i0; i < i1; ++i) {
      ssims[i] = m[3 * (i - i0)];
      psnrs[i] = m[3 * (i - i0) + 1];
      maes[i] = m[3 * (i - i0) + 2];
    }
    i0 = i1;
  }

  std::FILE* csv = nullptr;
  if (!csv_out.empty()) {
    csv = std::fopen(csv_out.string().c_str(), "w");
    if (!csv) throw HostError{TG_ERR_IO, "cannot write " + csv_out.string()};
    std::fprintf(csv, "object,position_index,depth_index,ssim,psnr_db,mae_pct\n");
    for (size_t i = 0; i < n; ++i)
      std::fprintf(csv, "%s,%d,%d,%.6f,%.4f,%.4f\n", std::get<0>(keys[i]).c_str(),
                   std::get<1>(keys[i]), std::get<2>(keys[i]), ssims[i], psnrs[i], maes[i]);
  }
  CompareAggregate agg;
  agg.pairs = n;
  auto mean = [](const std::vector<double>& xs) {
    double s = 0.0;
    for (double x : xs) s += x;
    return xs.empty() ? 0.0 : s / static_cast<double>(xs.size());
  };
  agg.ssim_mean = mean(ssims);
  agg.psnr_mean = mean(psnrs);
  agg.mae_mean = mean(maes);
  agg.ssim_std = aggregate_std(ssims, agg.ssim_mean);
  agg.psnr_std = aggregate_std(psnrs, agg.psnr_mean);
  agg.mae_std = aggregate_std(maes, agg.mae_mean);
  if (csv) {
    std::fprintf(csv, "mean,,,%.6f,%.4f,%.4f\n", agg.ssim_mean, agg.psnr_mean, agg.mae_mean);
    std::fprintf(csv, "std,,,%.6f,%.4f,%.4f\n", agg.ssim_std, agg.psnr_std, agg.mae_std);
    std::fclose(csv);
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
