// Test-side pin of the scene document layout. The reference serializes scenes with
// nlohmann::json (scene.cpp:472-556: doc.dump(2) + "\n"; vendor/json.hpp is not in
// /root/reference, the copy shipped with this image is used). This program parses
// stdin with nlohmann and prints dump(2) + "\n": for a document the product's
// serialize_scene wrote, the output must be the same bytes.
#include <iostream>
#include <sstream>

#include <nlohmann/json.hpp>

int main() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const nlohmann::json doc = nlohmann::json::parse(ss.str());
  std::cout << doc.dump(2) << "\n";
  return 0;
}
