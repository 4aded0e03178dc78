// File formats either side of the hot path (io.cu); see include/fm_gpu.h.
#pragma once

#include <string>

#include "../../include/fm_gpu.h"

namespace fmh {
void raster_read(const std::string& path, fm_raster* out);
void raster_release(fm_raster* r);
void raster_write_ascii(const fm_raster* r, const std::string& path);
void raster_write_bin(const fm_raster* r, const std::string& path);
void grid_write(const fm_grid* g, const std::string& path, bool binary);
void grid_read(const std::string& path, fm_grid** out);
}  // namespace fmh
