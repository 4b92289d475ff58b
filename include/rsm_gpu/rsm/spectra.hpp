// Forwarding header: the reference's <rsm/spectra.hpp> resolves to the B200
// drop-in (include/rsm_gpu/rsm.hpp) when include/rsm_gpu is on the include
// path ahead of the reference's headers.
#pragma once
#include "../rsm.hpp"
