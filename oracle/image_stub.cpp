// image_stub.cpp — TEST INFRASTRUCTURE ONLY.  libpng is absent here, so the
// reference's src/image.cpp cannot be built; io.cpp links against these
// stubs (read_image / write_image are not on the path under test).
#include <stdexcept>
#include <string>

#include "evsim/image.hpp"

namespace evsim {
ImageU8 read_image(const std::string& path) { throw std::runtime_error("'" + path + "': image I/O not built"); }
void write_image(const ImageU8&, const std::string& path) {
  throw std::runtime_error("'" + path + "': image I/O not built");
}
}  // namespace evsim
