#pragma once
// Drop-in path for the reference header rectri/gemm.hpp: the whole rectri API
// is provided by rectri_b200.hpp on top of the sm_100a library.
#include "../rectri_b200.hpp"
