// Launch-attribute switches shared by every kernel launcher.
#pragma once

namespace wm {
// Programmatic dependent launch on every kernel (default on; the "pdl" context
// option turns it off for measurements).
extern bool g_pdl;
}  // namespace wm
