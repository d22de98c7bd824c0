// Host file formats shared by the bridge (bridge.cpp) and the dataset harness
// (harness.cpp): PNG via zlib (render/image.cpp) and the .depth format
// (render/depth_map.cpp). References are to /root/reference/proj.
#include <zlib.h>

#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "host_config.hpp"
#include "tacchi_cuda.h"

namespace tacchi_b200::host {

using json = nlohmann::json;

namespace {

// ---- on-disk formats -------------------------------------------------------

uint32_t be32(uint32_t v) {
  return ((v & 0xffu) << 24) | ((v & 0xff00u) << 8) | ((v >> 8) & 0xff00u) | (v >> 24);
}

void png_chunk(std::ofstream& out, const char* type, const unsigned char* data, uint32_t len) {
  const uint32_t blen = be32(len);
  out.write(reinterpret_cast<const char*>(&blen), 4);
  out.write(type, 4);
  if (len) out.write(reinterpret_cast<const char*>(data), len);
  uLong crc = crc32(0L, reinterpret_cast<const Bytef*>(type), 4);
  if (len) crc = crc32(crc, data, len);
  const uint32_t bcrc = be32(static_cast<uint32_t>(crc));
  out.write(reinterpret_cast<const char*>(&bcrc), 4);
}

uint32_t rd32(const unsigned char* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
}

int paeth(int a, int b, int c) {
  const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

}  // namespace

// render::save_png (image.cpp:23-49): 8-bit RGB, non-interlaced.
void save_png(const std::string& path, int w, int h, const uint8_t* rgb) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw HostError{TG_ERR_IO, "cannot write " + path};
  static const unsigned char sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
  out.write(reinterpret_cast<const char*>(sig), 8);
  unsigned char ihdr[13];
  const uint32_t bw = be32(static_cast<uint32_t>(w)), bh = be32(static_cast<uint32_t>(h));
  std::memcpy(ihdr, &bw, 4);
  std::memcpy(ihdr + 4, &bh, 4);
  ihdr[8] = 8;   // bit depth
  ihdr[9] = 2;   // colour type RGB
  ihdr[10] = 0;  // compression
  ihdr[11] = 0;  // filter
  ihdr[12] = 0;  // interlace
  png_chunk(out, "IHDR", ihdr, 13);
  std::vector<unsigned char> raw(static_cast<size_t>(h) * (3 * w + 1));
  for (int r = 0; r < h; ++r) {
    raw[static_cast<size_t>(r) * (3 * w + 1)] = 0;  // filter: none
    std::memcpy(&raw[static_cast<size_t>(r) * (3 * w + 1) + 1], rgb + static_cast<size_t>(r) * 3 * w,
                3 * static_cast<size_t>(w));
  }
  uLongf zlen = compressBound(raw.size());
  std::vector<unsigned char> z(zlen);
  if (compress2(z.data(), &zlen, raw.data(), raw.size(), 6) != Z_OK)
    throw HostError{TG_ERR_IO, "png compression failed"};
  png_chunk(out, "IDAT", z.data(), static_cast<uint32_t>(zlen));
  png_chunk(out, "IEND", nullptr, 0);
}

// render::save_depth_map (depth_map.cpp:28-38): JSON header line + float32.
void save_depth_map(const std::string& path, int w, int h, double pixel_to_meter,
                    const double* values) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw HostError{TG_ERR_IO, "cannot write " + path};
  const json header = {{"width", w}, {"height", h}, {"pixel_to_meter", pixel_to_meter}};
  out << header.dump() << '\n';
  std::vector<float> buf(static_cast<size_t>(w) * h);
  for (size_t i = 0; i < buf.size(); ++i) buf[i] = static_cast<float>(values[i]);
  out.write(reinterpret_cast<const char*>(buf.data()),
            static_cast<std::streamsize>(buf.size() * sizeof(float)));
}

std::vector<uint8_t> load_png(const std::string& path, int& w, int& h) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw HostError{TG_ERR_IO, "cannot open " + path};
  const std::vector<unsigned char> d((std::istreambuf_iterator<char>(in)),
                                     std::istreambuf_iterator<char>());
  static const unsigned char sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
  auto bad = [&](const std::string& why) -> HostError {
    return HostError{TG_ERR_PARSE, "not a readable PNG: " + path + " (" + why + ")"};
  };
  if (d.size() < 8 || std::memcmp(d.data(), sig, 8) != 0) throw bad("signature");
  size_t pos = 8;
  int depth = 0, ctype = -1, interlace = 0;
  std::vector<unsigned char> idat, plte;
  while (pos + 12 <= d.size()) {
    const uint32_t n = rd32(&d[pos]);
    if (pos + 12 + n > d.size()) throw bad("truncated chunk");
    const unsigned char* body = &d[pos + 8];
    const std::string type(reinterpret_cast<const char*>(&d[pos + 4]), 4);
    if (type == "IHDR") {
      w = static_cast<int>(rd32(body));
      h = static_cast<int>(rd32(body + 4));
      depth = body[8];
      ctype = body[9];
      interlace = body[12];
    } else if (type == "PLTE") {
      plte.assign(body, body + n);
    } else if (type == "IDAT") {
      idat.insert(idat.end(), body, body + n);
    } else if (type == "IEND") {
      break;
    }
    pos += 12 + n;
  }
  if (w <= 0 || h <= 0 || ctype < 0) throw bad("missing IHDR");
  if (interlace != 0) throw bad("interlaced PNGs are not supported");
  int channels;
  switch (ctype) {
    case 0: channels = 1; break;
    case 2: channels = 3; break;
    case 3: channels = 1; break;
    case 4: channels = 2; break;
    case 6: channels = 4; break;
    default: throw bad("colour type");
  }
  if (!(depth == 8 || depth == 16 || (depth < 8 && (ctype == 0 || ctype == 3))))
    throw bad("bit depth");
  const size_t bits_pp = static_cast<size_t>(channels) * depth;
  const size_t stride = (static_cast<size_t>(w) * bits_pp + 7) / 8;
  const size_t bpp = std::max<size_t>(1, bits_pp / 8);
  std::vector<unsigned char> raw(static_cast<size_t>(h) * (stride + 1));
  uLongf raw_len = raw.size();
  if (uncompress(raw.data(), &raw_len, idat.data(), idat.size()) != Z_OK || raw_len != raw.size())
    throw bad("inflate");
  std::vector<unsigned char> img(static_cast<size_t>(h) * stride), prev(stride, 0);
  for (int r = 0; r < h; ++r) {  // PNG filters (RFC 2083 6)
    const unsigned char ft = raw[r * (stride + 1)];
    const unsigned char* line = &raw[r * (stride + 1) + 1];
    unsigned char* cur = &img[r * stride];
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= bpp ? cur[i - bpp] : 0, b = prev[i], c = i >= bpp ? prev[i - bpp] : 0;
      int p = 0;
      switch (ft) {
        case 0: p = 0; break;
        case 1: p = a; break;
        case 2: p = b; break;
        case 3: p = (a + b) / 2; break;
        case 4: p = paeth(a, b, c); break;
        default: throw bad("filter type");
      }
      cur[i] = static_cast<unsigned char>(line[i] + p);
    }
    std::memcpy(prev.data(), cur, stride);
  }
  // png_set_expand / strip_16 / strip_alpha / gray_to_rgb (image.cpp:71-75)
  std::vector<uint8_t> rgb(static_cast<size_t>(w) * h * 3);
  for (int r = 0; r < h; ++r) {
    const unsigned char* row = &img[r * stride];
    for (int x = 0; x < w; ++x) {
      auto sample = [&](int ch) -> int {  // 8-bit value of channel ch
        if (depth == 16) return row[(static_cast<size_t>(x) * channels + ch) * 2];
        if (depth == 8) return row[static_cast<size_t>(x) * channels + ch];
        const size_t bit = static_cast<size_t>(x) * depth;
        const int v = (row[bit / 8] >> (8 - depth - bit % 8)) & ((1 << depth) - 1);
        return ctype == 3 ? v : v * 255 / ((1 << depth) - 1);
      };
      uint8_t* o = &rgb[(static_cast<size_t>(r) * w + x) * 3];
      if (ctype == 3) {
        const int idx = sample(0);
        if (static_cast<size_t>(3 * idx + 2) >= plte.size()) throw bad("palette index");
        o[0] = plte[3 * idx];
        o[1] = plte[3 * idx + 1];
        o[2] = plte[3 * idx + 2];
      } else if (ctype == 0 || ctype == 4) {
        o[0] = o[1] = o[2] = static_cast<uint8_t>(sample(0));
      } else {
        o[0] = static_cast<uint8_t>(sample(0));
        o[1] = static_cast<uint8_t>(sample(1));
        o[2] = static_cast<uint8_t>(sample(2));
      }
    }
  }
  return rgb;
}

}  // namespace tacchi_b200::host
