// Drop-in path of the reference header of the same name; the whole API is in tencache.hpp.
#pragma once
#include "tencache/tencache.hpp"
