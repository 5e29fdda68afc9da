// Drop-in for the reference header tslb/bench.hpp: the B200-backed interface
// lives in one header (see tslb_b200/tslb.hpp for the mapping).
#pragma once
#include "../tslb_b200/tslb.hpp"
