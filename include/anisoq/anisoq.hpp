// anisoq drop-in (B200): umbrella header (reference anisoq.hpp). Compile with
// -I <repo>/include and link <repo>/paper_1908_10396_b200/libanisoq_b200.so.
#pragma once

#include "dataset.hpp"
#include "error.hpp"
#include "geometry.hpp"
#include "index.hpp"
#include "parallel.hpp"
#include "pq.hpp"
#include "rng.hpp"
#include "vq.hpp"
