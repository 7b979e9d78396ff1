// Drop-in include path (#include "pcadmm/bignat.hpp"): BigNat / Rng of the B200 facade.
#pragma once
#include "../../pcb200_pcadmm.hpp"
