// Reference-compatible include path (perfseer/manifest.hpp); declarations in
// ps_manifest.hpp.
#pragma once
#include "../ps_manifest.hpp"
