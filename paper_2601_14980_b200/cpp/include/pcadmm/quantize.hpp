// Drop-in include path (#include "pcadmm/quantize.hpp"): the B200 quantizer API.
#pragma once
#include "../../pcb200_quantize.hpp"
